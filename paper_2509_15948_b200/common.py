"""Shared constants and seeding helpers.

Restates ``mg/common.py:7-22``: the whole path is hard-wired to a 30 kHz
sample clock, and every random draw comes from a named substream of a root
seed so that stems, parameter inits and reverb noise are byte-identical to
the reference's.
"""

from __future__ import annotations

import zlib

import numpy as np

SAMPLE_RATE = 30_000  # mg/common.py:7


def rng_for(seed: int, label: str) -> np.random.Generator:
    """Named RNG substream (mg/common.py:10-13): SeedSequence([seed, crc32(label)])."""
    return np.random.default_rng(
        np.random.SeedSequence([int(seed), zlib.crc32(label.encode("utf-8"))]))


def round_half_away(x: float) -> int:
    """Round half away from zero (mg/common.py:16-18)."""
    if x == 0:
        return 0
    return int(np.floor(abs(x) + 0.5) * np.sign(x))


def seconds_to_samples(t: float, sr: int = SAMPLE_RATE) -> int:
    """mg/common.py:21-22 (Python round, i.e. half-to-even)."""
    return int(round(t * sr))

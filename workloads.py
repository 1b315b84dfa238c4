"""Synthetic workloads for the bench and the tests (input data, not product code).

The reference's stem generator (``mg/synth.py:34-115``: ``SynthSpec``,
``make_stems``) restated byte-identically so that the bench and the parity
tests feed the device path exactly the stems the reference would generate for
a seed (``tests/test_reference_api.py`` pins it against the reference).  Stems
are round-tripped through float32 as ``mg/synth.py:217`` does.  It lives
outside the ``paper_2509_15948_b200`` package: input generation is out of the
hot path's scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2509_15948_b200.common import SAMPLE_RATE, rng_for
from paper_2509_15948_b200.console import SessionManifest, TrackEntry

STEM_KINDS = ("tonal", "noise", "percussive")


@dataclass
class SynthSpec:
    tracks: int = 4
    subgroups: int = 2
    duration_seconds: float = 10.0
    planted_fraction: float = 0.4
    stem_level: float = 0.35
    full_wet: bool = False


def _envelope(rng, n, sr):
    t = np.arange(n) / sr
    rate, duty, phase = rng.uniform(0.8, 3.0), rng.uniform(0.4, 0.8), rng.uniform(0, 1)
    env = 0.4 + 0.6 * (((t * rate + phase) % 1.0) < duty).astype(np.float64)
    ramp = np.ones(n)
    edge = min(n, int(0.004 * sr))
    ramp[:edge] = np.linspace(0, 1, edge)
    return env * ramp


def _tonal(rng, n, sr):
    t = np.arange(n) / sr
    f0 = rng.uniform(70, 900)
    sig = np.zeros(n)
    for h in range(1, 5):
        amp = rng.uniform(0.2, 1.0) / h
        vib = 1.0 + 0.002 * np.sin(2 * np.pi * rng.uniform(3, 7) * t)
        sig += amp * np.sin(2 * np.pi * f0 * h * vib * t + rng.uniform(0, 2 * np.pi))
    return sig


def _noise(rng, n, sr):
    white = rng.standard_normal(n + 512)
    lo, hi = sorted(rng.uniform(60, 12_000, size=2))
    spec = np.fft.rfft(white)
    freqs = np.fft.rfftfreq(white.size, d=1.0 / sr)
    spec[~((freqs >= lo) & (freqs <= max(hi, lo * 2)))] *= 0.02
    return np.fft.irfft(spec, n=white.size)[:n]


def _percussive(rng, n, sr):
    sig = np.zeros(n)
    period = int(sr / rng.uniform(1.5, 4.0))
    decay = np.exp(-np.arange(period) / (sr * rng.uniform(0.02, 0.08)))
    for start in range(int(rng.uniform(0, period / 2)), n, period):
        burst = rng.standard_normal(min(period, n - start))
        sig[start:start + burst.size] += burst * decay[:burst.size]
    return sig


_BUILD = {"tonal": _tonal, "noise": _noise, "percussive": _percussive}


def make_stems(spec: SynthSpec, seed):
    """(K, 2, n) float64 stems + kinds (mg/synth.py:93-115)."""
    n = int(round(spec.duration_seconds * SAMPLE_RATE))
    stems = np.zeros((spec.tracks, 2, n))
    kinds = []
    for k in range(spec.tracks):
        rng = rng_for(seed, f"stem-{k}")
        kind = STEM_KINDS[int(rng.integers(0, len(STEM_KINDS)))]
        kinds.append(kind)
        sig = _BUILD[kind](rng, n, SAMPLE_RATE) * _envelope(rng, n, SAMPLE_RATE)
        sig /= max(np.max(np.abs(sig)), 1e-9)
        lag = int(rng.integers(4, 24))
        lagged = np.concatenate([np.zeros(lag), sig[:-lag]])
        mix = rng.uniform(0.04, 0.1)
        stems[k, 0] = sig + 8e-3 * rng.standard_normal(n)
        stems[k, 1] = (1 - mix) * sig + mix * lagged + 8e-3 * rng.standard_normal(n)
        stems[k] *= spec.stem_level / max(np.sqrt(np.mean(stems[k] ** 2)), 1e-9)
    return stems, kinds


def make_stems_f32(spec: SynthSpec, seed, length=None):
    """Stems round-tripped through float32 (mg/synth.py:217), optionally cut to ``length``."""
    stems, _ = make_stems(spec, seed)
    stems = stems.astype(np.float32)
    return stems[..., :length] if length is not None else stems


def manifest_for(spec: SynthSpec):
    """Round-robin subgroup assignment ``groups[k % S]`` (mg/synth.py:211-214)."""
    groups = [f"bus{j}" for j in range(spec.subgroups)]
    tracks = [TrackEntry(f"stems/track{k:02d}.wav", f"track{k:02d}", groups[k % spec.subgroups])
              for k in range(spec.tracks)]
    return SessionManifest(tracks, "target.wav")

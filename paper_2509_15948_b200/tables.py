"""Host-built constant tables uploaded once per device.

* reverb noise STFTs and the OLA normaliser (recipe of mg/processors.py:127-145):
  uniform(-1, 1) noise of 60000 samples from the ``reverb-mid`` / ``reverb-side``
  substreams of seed 0x5EED0001, reflect-padded by 192, 313 frames x periodic
  Hann(384), rfft;
* the A-weighted HTK mel projection per FFT size (mg/losses.py:51-101), stored
  as band CSR (forward) and bin CSC (backward) because every band is a
  contiguous run of bins.
"""

from __future__ import annotations

import functools

import numpy as np

from .common import SAMPLE_RATE, rng_for

REVERB_NFFT, REVERB_HOP, REVERB_LEN = 384, 192, 60_000
REVERB_NOISE_SEED = 0x5EED_0001


def hann_periodic(n):
    return 0.5 - 0.5 * np.cos(2 * np.pi * np.arange(n) / n)


@functools.lru_cache(maxsize=None)
def reverb_tables():
    """(specs (2, 313, 193) complex128 [mid, side], wss (60000,), n_frames)."""
    win = hann_periodic(REVERB_NFFT)
    pad = REVERB_HOP
    n_frames = 1 + (REVERB_LEN + 2 * pad - REVERB_NFFT) // REVERB_HOP
    idx = np.arange(n_frames)[:, None] * REVERB_HOP + np.arange(REVERB_NFFT)[None, :]
    specs = []
    for chan in ("mid", "side"):
        noise = rng_for(REVERB_NOISE_SEED, f"reverb-{chan}").uniform(-1, 1, REVERB_LEN)
        specs.append(np.fft.rfft(np.pad(noise, pad, mode="reflect")[idx] * win, axis=-1))
    cover = (n_frames - 1) * REVERB_HOP + REVERB_NFFT
    wss = np.zeros(cover)
    for m in range(n_frames):
        wss[m * REVERB_HOP:m * REVERB_HOP + REVERB_NFFT] += win * win
    return np.stack(specs), wss[pad:pad + REVERB_LEN].copy(), n_frames


def _hz_to_mel(f):
    return 2595.0 * np.log10(1.0 + np.asarray(f, dtype=np.float64) / 700.0)


def _mel_to_hz(m):
    return 700.0 * (10.0 ** (np.asarray(m, dtype=np.float64) / 2595.0) - 1.0)


@functools.lru_cache(maxsize=None)
def mel_filterbank(n_fft, sr=SAMPLE_RATE, n_mels=96, fmax=15_000.0):
    """(n_mels, bins) HTK triangles with degenerate-band repair (mg/losses.py:51-73)."""
    freqs = np.fft.rfftfreq(n_fft, d=1.0 / sr)
    pts = _mel_to_hz(np.linspace(_hz_to_mel(0.0), _hz_to_mel(fmax), n_mels + 2))
    lo, pk, hi = pts[:-2, None], pts[1:-1, None], pts[2:, None]
    up = (freqs[None, :] - lo) / np.maximum(pk - lo, 1e-12)
    dn = (hi - freqs[None, :]) / np.maximum(hi - pk, 1e-12)
    fb = np.clip(np.minimum(up, dn), 0.0, None)
    for j in np.where(fb.sum(axis=1) == 0)[0]:
        fb[j, np.argmin(np.abs(freqs - pts[j + 1]))] = 1.0
    for k in np.where((freqs < sr / 2) & (fb.sum(axis=0) == 0))[0]:
        fb[np.argmin(np.abs(pts[1:-1] - freqs[k])), k] = 1.0
    return fb


@functools.lru_cache(maxsize=None)
def a_weight_gains(n_fft, sr=SAMPLE_RATE):
    f2 = np.fft.rfftfreq(n_fft, d=1.0 / sr) ** 2
    ra = (12194.0 ** 2 * f2 ** 2) / ((f2 + 20.6 ** 2) * np.sqrt((f2 + 107.7 ** 2) * (f2 + 737.9 ** 2))
                                     * (f2 + 12194.0 ** 2))
    return ra * 10.0 ** (2.0 / 20.0)


def projection(n_fft, sr, n_mels, fmax, a_weighting):
    """(bins, n_mels) A-weight x mel matrix (mg/losses.py:94-101)."""
    proj = mel_filterbank(n_fft, sr, n_mels, fmax).T.copy()
    if a_weighting:
        proj *= a_weight_gains(n_fft, sr)[:, None]
    return proj


@functools.lru_cache(maxsize=None)
def projection_sparse(n_fft, sr, n_mels, fmax, a_weighting):
    """Band CSR (start, len, off, w) and bin CSC (start, len, band, w) of the projection.

    Bands are stored over their full [first nonzero, last nonzero] bin range, so
    the banded product equals the dense ``|X| @ proj`` term for term."""
    P = projection(n_fft, sr, n_mels, fmax, a_weighting)
    bins = P.shape[0]
    b_start, b_len, b_off, b_w = [], [], [], []
    off = 0
    for j in range(n_mels):
        nz = np.nonzero(P[:, j])[0]
        k0, k1 = (int(nz[0]), int(nz[-1]) + 1) if nz.size else (0, 0)
        b_start.append(k0)
        b_len.append(k1 - k0)
        b_off.append(off)
        b_w.extend(P[k0:k1, j].tolist())
        off += k1 - k0
    c_start, c_len, c_band, c_w = [], [], [], []
    for k in range(bins):
        nz = np.nonzero(P[k, :])[0]
        c_start.append(len(c_band))
        c_len.append(len(nz))
        c_band.extend(nz.tolist())
        c_w.extend(P[k, nz].tolist())
    i32 = lambda a: np.asarray(a, dtype=np.int32)  # noqa: E731
    return (i32(b_start), i32(b_len), i32(b_off), np.asarray(b_w, dtype=np.float64),
            i32(c_start), i32(c_len), i32(c_band), np.asarray(c_w, dtype=np.float64))

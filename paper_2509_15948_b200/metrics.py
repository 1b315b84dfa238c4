"""Post-hoc song metrics on the device (mg/metrics.py:45-112; mg/cli.py:42-63).

Once a search ends, the reference renders the final graph over the whole
session (the "match", mg/cli.py:42-45) and scores it against the target:
the audio loss L_a, the scale-invariant SDR, and the log10 mean-squared
distance of five per-segment MIR features (RMS, crest factor, stereo width,
stereo imbalance, Bark-band log spectrum) over 8-second segments.  Here the
match is rendered by the device path and every metric is reduced by
``mgb_song_metrics`` (float64 sums over float32 signals; the Bark spectrum's
240,000-point rfft by Bluestein on the library's power-of-two FFT).
"""

from __future__ import annotations

import numpy as np
import torch

from ._lib import check, lib
from .common import SAMPLE_RATE
from .engine import F32, F64, ensure_device, ptr, stream_ptr

SEGMENT_SECONDS = 8.0
FLOOR = 1e-12
BARK_EDGES = np.array([0, 100, 200, 300, 400, 510, 630, 770, 920, 1080, 1270, 1480, 1720, 2000, 2320, 2700, 3150,
                       3700, 4400, 5300, 6400, 7720, 9500, 12000, 15000], dtype=np.float64)
FEATURES = ("rms", "cf", "sw", "si", "bs")


class TooShort(Exception):
    pass


class ZeroTarget(Exception):
    pass


def _stats(y, y_hat, device):
    dev = ensure_device(device)
    yt = torch.as_tensor(np.asarray(y) if not torch.is_tensor(y) else y).to(dev, F32).contiguous()
    ht = torch.as_tensor(np.asarray(y_hat) if not torch.is_tensor(y_hat) else y_hat).to(dev, F32).contiguous()
    if yt.shape != ht.shape or yt.dim() != 2 or yt.shape[0] != 2:
        raise ZeroTarget(f"length mismatch {tuple(yt.shape)} vs {tuple(ht.shape)}")
    L = int(yt.shape[-1])
    seg = int(round(SEGMENT_SECONDS * SAMPLE_RATE))
    nseg = L // seg
    Ld = lib()
    ws_bytes = int(Ld.mgb_metrics_workspace(L, seg))
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
    nb = BARK_EDGES.size - 1
    edges = torch.from_numpy(BARK_EDGES).to(dev)
    stats = torch.zeros((max(nseg, 1), 10), dtype=F64, device=dev)
    dots = torch.zeros(5, dtype=F64, device=dev)
    by = torch.zeros((max(nseg, 1), nb), dtype=F64, device=dev)
    bh = torch.zeros_like(by)
    check(Ld.mgb_song_metrics(ptr(yt), ptr(ht), L, seg, ptr(edges), nb, float(SAMPLE_RATE), ptr(stats), ptr(dots),
                              ptr(by), ptr(bh), ptr(ws), ws_bytes, stream_ptr()), "mgb_song_metrics")
    return nseg, seg, stats.cpu().numpy(), dots.cpu().numpy(), by.cpu().numpy(), bh.cpu().numpy()


def _features(nseg, seg, stats, by, bh):
    """Per signal (0 = target, 1 = match): feature -> (segments, k) array."""
    out = []
    for w in range(2):
        s = stats[:nseg, 5 * w:5 * w + 5]
        mid2, mx, side2, el, er = (s[:, i] for i in range(5))
        rms = np.sqrt(mid2 / seg)
        out.append({
            "rms": rms[:, None],
            "cf": (mx / np.maximum(rms, FLOOR))[:, None],
            "sw": (side2 / np.maximum(mid2, FLOOR))[:, None],
            "si": ((er - el) / np.maximum(er + el, FLOOR))[:, None],
            "bs": (by if w == 0 else bh)[:nseg],
        })
    return out


def si_sdr_from(dots, cap_db=100.0):
    ss, _, _, num, den = (float(v) for v in dots)
    if ss == 0.0:
        raise ZeroTarget("target signal is identically zero")
    if den == 0.0 or num / den > 10 ** (cap_db / 10):
        return cap_db
    return float(10 * np.log10(num / den))


def mir_distances(y, y_hat, device="cuda"):
    """{feature: log10 of the per-segment feature MSE} for every feature (mg/metrics.py:85-93)."""
    nseg, seg, stats, _, by, bh = _stats(y, y_hat, device)
    if nseg < 1:
        raise TooShort(f"need at least {seg} samples, got {np.shape(y)[-1]}")
    fy, fh = _features(nseg, seg, stats, by, bh)
    out = {}
    for f in FEATURES:
        k = fy[f].shape[1]
        total = float(np.sum((fy[f] - fh[f]) ** 2))
        out[f] = float(np.log10(max(total / (nseg * k), FLOOR)))
    return out


def mir_distance(y, y_hat, feature, device="cuda"):
    return mir_distances(y, y_hat, device)[feature]


def si_sdr(y, y_hat, cap_db=100.0, device="cuda"):
    """Scale-invariant SDR over the concatenated stereo channels, in dB (mg/metrics.py:96-112)."""
    return si_sdr_from(_stats(y, y_hat, device)[3], cap_db)


def song_metrics(name, target, match, warmup_len, loss_cfg=None, device="cuda"):
    """The reference's per-song metrics row (mg/cli.py:55-63) for a rendered match:
    L_a, si_sdr and d_<feature> (empty string where a feature is undefined)."""
    from .losses import LossConfig, mrstft
    loss_cfg = loss_cfg or LossConfig()
    dev = ensure_device(device)
    mt = torch.as_tensor(np.asarray(match) if not torch.is_tensor(match) else match).to(dev, F32)
    tg = torch.as_tensor(np.asarray(target) if not torch.is_tensor(target) else target).to(dev, F32)
    la = float(mrstft(mt[:, warmup_len:].contiguous(), tg[:, warmup_len:].contiguous(), loss_cfg))
    nseg, seg, stats, dots, by, bh = _stats(tg, mt, dev)
    row = {"name": name, "L_a": la, "si_sdr": si_sdr_from(dots)}
    if nseg >= 1:
        fy, fh = _features(nseg, seg, stats, by, bh)
        for f in FEATURES:
            total = float(np.sum((fy[f] - fh[f]) ** 2))
            row[f"d_{f}"] = float(np.log10(max(total / (nseg * fy[f].shape[1]), FLOOR)))
    else:
        for f in FEATURES:
            row[f"d_{f}"] = ""
    return row


def render_match(graph, params, stems, device="cuda"):
    """The final graph rendered over the whole session (mg/cli.py:42-45), on the device."""
    from .scheduler import execute_batched
    from .schedule import schedule_for
    y, _ = execute_batched(graph, params, stems, schedule_for(graph), device=device)
    return y


__all__ = ["FEATURES", "mir_distance", "mir_distances", "si_sdr", "song_metrics", "render_match", "TooShort",
           "ZeroTarget"]

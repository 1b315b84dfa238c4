"""Per-type processor kernels on the device, with the reference's call shape.

``KERNELS[tag](u, p) -> (ybar, reg | None)`` mirrors ``mg/processors.py:321-329``:
``u`` is a (B, 2, L) float32 CUDA tensor (or anything torch.as_tensor accepts),
``p`` the (B, N_t) parameter rows (float64).  The call runs the level kernel
with the dry/wet disabled (``w = NULL``) and is differentiable through torch
autograd: its backward is the level's hand-written adjoint
(``mgb_level_backward``), the device counterpart of the reference tape's
replay (``mg/engine.py:100-112``).  ``drywet_wrap`` and ``gain_staging_term``
are exposed for API parity; the engine itself fuses both into the level
kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import MgbLevel, check, lib
from .engine import F32, F64, I32, dev_ptr_array, ensure_device, ptr, stream_ptr
from .graph import PARAM_COUNTS

EQ_FIR_LEN, EQ_BINS = 2047, 1024
REVERB_NFFT, REVERB_HOP, REVERB_PARAM_BINS = 384, 192, 192
REVERB_NOISE_LEN = 60_000
BALLISTICS_LEN, ENVELOPE_EPS = 8192, 1e-8
DELAY_TAPS, DELAY_WINDOW, COLOR_LEN, COLOR_BINS = 20, 3000, 39, 20
DELAY_FIR_LEN = DELAY_TAPS * DELAY_WINDOW + COLOR_LEN - 1
DELAY_RADIUS_GAMMA = 0.01
GAIN_STAGING_EPS = 1e-8


def _as_u(u, device=None):
    t = u if torch.is_tensor(u) else torch.as_tensor(np.asarray(u))
    dev = ensure_device(device or (t.device if t.is_cuda else "cuda"))
    t = t.to(device=dev, dtype=F32).contiguous()
    if t.data_ptr() % 16:  # the level kernels use 16-byte vector loads on rows when L % 4 == 0
        t = t.clone()
    return t


class _Level:
    """Single-level device state for one KERNELS call (rows = the batch)."""

    def __init__(self, tag, u, p):
        dev = u.device
        B, _, L = u.shape
        self.tag, self.B, self.L = tag, B, L
        self.u, self.p = u, p
        Ld = lib()
        self.rows = dev_ptr_array([ptr(u, b * 2 * L) for b in range(B)], dev)
        self.prow = torch.arange(B, dtype=I32, device=dev)
        self.widx = torch.arange(B, dtype=I32, device=dev)
        self.ws_bytes = int(Ld.mgb_level_workspace(tag.encode(), B, L))
        self.ws = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8, device=dev)
        self.y = torch.empty((B, 2, L), dtype=F32, device=dev)
        self.ybar = torch.empty((B, 2, L), dtype=F32, device=dev) if tag in "erd" else None
        self.aux = torch.empty((B, L), dtype=F32, device=dev) if tag in "cn" else None
        self.reg = torch.zeros(B, dtype=F64, device=dev)

    def struct(self):
        s = MgbLevel()
        s.tag = self.tag.encode()
        s.B, s.L = self.B, self.L
        s.u_rows, s.bank = ptr(self.rows), ptr(self.p)
        s.prow, s.widx = ptr(self.prow), ptr(self.widx)
        s.w = None
        s.y = ptr(self.y)
        s.ybar = ptr(self.ybar) if self.ybar is not None else None
        s.aux = ptr(self.aux) if self.aux is not None else None
        s.reg = ptr(self.reg)
        s.ws, s.ws_bytes = ptr(self.ws), self.ws_bytes
        return s


class _KernelFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, tag, u, p):
        lv = _Level(tag, u, p)
        st = lv.struct()
        check(lib().mgb_level_forward(ctypes.byref(st), stream_ptr()), f"{tag} forward")
        ctx.lv = lv
        out = lv.ybar if lv.ybar is not None else lv.y
        return out, lv.reg.sum()

    @staticmethod
    def backward(ctx, gy, greg):
        lv = ctx.lv
        B, L = lv.B, lv.L
        gy = (gy if gy is not None else torch.zeros_like(lv.y)).to(F32).contiguous()
        if gy.data_ptr() % 16:
            gy = gy.clone()
        gyr = dev_ptr_array([ptr(gy, b * 2 * L) for b in range(B)], gy.device)
        greg_t = (greg if greg is not None else torch.zeros((), device=gy.device)).to(F64).reshape(())
        gu = torch.empty((B, 2, L), dtype=F32, device=gy.device)
        gp = torch.zeros_like(lv.p)
        gw = torch.zeros(B, dtype=F64, device=gy.device)
        st = lv.struct()
        st.gy_rows, st.greg = ptr(gyr), ptr(greg_t)
        st.gu, st.gbank, st.gw = ptr(gu), ptr(gp), ptr(gw)
        check(lib().mgb_level_backward(ctypes.byref(st), stream_ptr()), f"{lv.tag} backward")
        return None, gu, gp


def _kernel(tag):
    def run(u, p):
        ut = _as_u(u)
        pt = p if torch.is_tensor(p) else torch.as_tensor(np.asarray(p, dtype=np.float64))
        pt = pt.to(device=ut.device, dtype=F64)
        if pt.dim() != 2 or pt.shape[1] != PARAM_COUNTS[tag] or pt.shape[0] != ut.shape[0]:
            raise ValueError(f"{tag}: expected p of shape ({ut.shape[0]}, {PARAM_COUNTS[tag]})")
        ybar, reg = _KernelFn.apply(tag, ut, pt.contiguous())
        return ybar, (reg if tag in "erd" else None)
    run.__name__ = {"g": "gain_panning", "s": "stereo_imager", "e": "equalizer", "r": "reverb",
                    "c": "compressor", "n": "noisegate", "d": "multitap_delay"}[tag]
    return run


KERNELS = {t: _kernel(t) for t in "gsercnd"}
gain_panning, stereo_imager = KERNELS["g"], KERNELS["s"]
equalizer, reverb = KERNELS["e"], KERNELS["r"]
compressor, noisegate, multitap_delay = KERNELS["c"], KERNELS["n"], KERNELS["d"]


def drywet_wrap(kernel_out, u, w):
    """w * wet + (1 - w) * u, exactly u where w == 0 (mg/processors.py:61-73)."""
    w = torch.as_tensor(w, dtype=F64, device=kernel_out.device).reshape(-1, 1, 1)
    mixed = (w * kernel_out + (1.0 - w) * u).to(kernel_out.dtype)
    return torch.where((w == 0).expand_as(u), u, mixed)


def gain_staging_term(u, ybar):
    """sum_b |log ||wet_mid|| - log ||in_mid||| (mg/processors.py:83-90)."""
    nu = torch.linalg.vector_norm((u[:, 0] + u[:, 1]).to(F64), dim=-1)
    ny = torch.linalg.vector_norm((ybar[:, 0] + ybar[:, 1]).to(F64), dim=-1)
    return torch.sum(torch.abs(torch.log(ny + GAIN_STAGING_EPS) - torch.log(nu + GAIN_STAGING_EPS)))


def quantize_delay(z):
    """Host helper with the reference's float64 semantics (mg/processors.py:250-254)."""
    pos = (-np.angle(z)) % (2 * np.pi) / (2 * np.pi) * DELAY_WINDOW
    return np.rint(pos).astype(int) % DELAY_WINDOW

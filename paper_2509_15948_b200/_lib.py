"""ctypes binding of libmixgraph_b200.so (the C ABI in include/mixgraph_b200.h).

The library is built in-tree for sm_100a (``__graft_entry__.build()`` or
``make -C paper_2509_15948_b200/csrc``).  There is no fallback: if the shared
object is missing or fails to load, every device entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmixgraph_b200.so")

c_void_p, c_int, c_size_t, c_double, c_float, c_char, c_longlong = (
    ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_double, ctypes.c_float,
    ctypes.c_char, ctypes.c_longlong)


class MgbLevel(ctypes.Structure):
    _fields_ = [
        ("tag", c_char), ("B", c_int), ("L", c_int),
        ("u_rows", c_void_p), ("gy_rows", c_void_p),
        ("bank", c_void_p), ("prow", c_void_p), ("widx", c_void_p),
        ("w", c_void_p), ("greg", c_void_p),
        ("y", c_void_p), ("ybar", c_void_p), ("aux", c_void_p), ("reg", c_void_p),
        ("gu", c_void_p), ("gbank", c_void_p), ("gw", c_void_p),
        ("ws", c_void_p), ("ws_bytes", c_size_t),
    ]


class MgbLossRes(ctypes.Structure):
    _fields_ = [
        ("n_fft", c_int), ("hop", c_int), ("frames", c_int), ("n_mels", c_int),
        ("band_start", c_void_p), ("band_len", c_void_p), ("band_off", c_void_p), ("band_w", c_void_p),
        ("bin_start", c_void_p), ("bin_len", c_void_p), ("bin_band", c_void_p), ("bin_w", c_void_p),
        ("tmel", c_void_p), ("tlog", c_void_p), ("mel", c_void_p), ("part", c_void_p),
        ("gframes", c_void_p),
    ]


class MgbLoss(ctypes.Structure):
    _fields_ = [
        ("n_res", c_int), ("res", MgbLossRes * 8), ("Ls", c_int),
        ("group_w", c_double * 4), ("stats", c_void_p), ("loss", c_void_p),
        ("batch", c_int), ("sig_stride", c_longlong),
    ]


class LibraryMissing(RuntimeError):
    pass


class DeviceError(RuntimeError):
    pass


_lib = None
ABI_VERSION = 4  # MGB_ABI_VERSION in include/mixgraph_b200.h


def lib():
    """Load (once) and return the shared library; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} is not built; run __graft_entry__.build() "
            "(nvcc, sm_100a). There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    L.mgb_abi_version.restype = c_int
    if L.mgb_abi_version() != ABI_VERSION:
        raise LibraryMissing(f"{LIB_PATH} has ABI {L.mgb_abi_version()}, this binding needs {ABI_VERSION}; "
                             "rebuild it (__graft_entry__.build())")
    L.mgb_init.argtypes = [c_void_p, c_void_p, c_void_p]
    L.mgb_level_workspace.argtypes = [c_char, c_int, c_int]
    L.mgb_level_workspace.restype = c_size_t
    L.mgb_level_forward.argtypes = [ctypes.POINTER(MgbLevel), c_void_p]
    L.mgb_level_backward.argtypes = [ctypes.POINTER(MgbLevel), c_void_p]
    L.mgb_level_forward_phase.argtypes = [ctypes.POINTER(MgbLevel), c_int, c_void_p]
    L.mgb_level_backward_phase.argtypes = [ctypes.POINTER(MgbLevel), c_int, c_void_p]
    L.mgb_launch_count.restype = c_longlong
    L.mgb_launch_count.argtypes = []
    L.mgb_weights.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_void_p]
    L.mgb_bus_sum.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p]
    L.mgb_fft.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_float, c_void_p]
    L.mgb_mrstft_target.argtypes = [ctypes.POINTER(MgbLoss), c_void_p, c_void_p, c_void_p]
    L.mgb_mrstft_forward.argtypes = [ctypes.POINTER(MgbLoss), c_void_p, c_void_p, c_void_p]
    L.mgb_mrstft_backward.argtypes = [ctypes.POINTER(MgbLoss), c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p]
    L.mgb_adamw_step.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_longlong, c_longlong, c_int,
                                 c_longlong, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_void_p]
    L.mgb_sparsity.argtypes = [c_void_p, c_int, c_void_p, c_void_p]
    L.mgb_gather_rows.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p]
    L.mgb_zero.argtypes = [c_void_p, c_size_t, c_void_p]
    L.mgb_timestamp.argtypes = [c_void_p, c_void_p]
    L.mgb_loss_assembly.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_int,
                                    c_void_p, c_void_p, c_void_p]
    L.mgb_metrics_workspace.argtypes = [c_int, c_int]
    L.mgb_metrics_workspace.restype = c_size_t
    L.mgb_song_metrics.argtypes = [c_void_p, c_void_p, c_int, c_int, c_void_p, c_int, c_double, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]
    L.mgb_stream_create.argtypes = []
    L.mgb_stream_create.restype = c_void_p
    L.mgb_stream_create_priority.argtypes = [c_int]
    L.mgb_stream_create_priority.restype = c_void_p
    L.mgb_stream_destroy.argtypes = [c_void_p]
    for name in ("mgb_init", "mgb_level_forward", "mgb_level_backward", "mgb_level_forward_phase",
                 "mgb_level_backward_phase", "mgb_weights", "mgb_bus_sum",
                 "mgb_fft", "mgb_mrstft_target", "mgb_mrstft_forward", "mgb_mrstft_backward",
                 "mgb_adamw_step", "mgb_sparsity", "mgb_stream_destroy", "mgb_gather_rows", "mgb_song_metrics", "mgb_loss_assembly", "mgb_zero", "mgb_timestamp"):
        getattr(L, name).restype = c_int
    _lib = L
    return L


EXPORTED = ("mgb_abi_version", "mgb_init", "mgb_level_workspace", "mgb_level_forward",
            "mgb_level_backward", "mgb_level_forward_phase", "mgb_level_backward_phase", "mgb_launch_count", "mgb_weights", "mgb_bus_sum", "mgb_fft", "mgb_mrstft_target",
            "mgb_mrstft_forward", "mgb_mrstft_backward", "mgb_adamw_step", "mgb_sparsity",
            "mgb_stream_create", "mgb_stream_destroy", "mgb_stream_create_priority", "mgb_gather_rows", "mgb_metrics_workspace",
            "mgb_song_metrics", "mgb_loss_assembly", "mgb_zero", "mgb_timestamp")


def check(rc, what):
    if rc != 0:
        raise DeviceError(f"{what} failed with status {rc}")

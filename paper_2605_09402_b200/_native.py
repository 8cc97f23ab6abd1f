"""ctypes binding of libatlas_b200.so (include/atlas_b200.h).

The library is built in-tree for sm_100a (``__graft_entry__.build()`` or
``make -C paper_2605_09402_b200/csrc``). There is no CPU fallback: if the
library or a CUDA device is missing, ``lib()`` raises DeviceError.
"""

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import DeviceError, IncompleteLayerError, raise_for_status

LIB_PATH = Path(__file__).resolve().parent / os.environ.get(
    "ATLAS_LIB", "libatlas_b200.so")  # ATLAS_LIB: A/B builds (diagnostics)

GCN, SAGE, GIN, GAT = 0, 1, 2, 3
F32, F16, BF16 = 0, 1, 2
MINPEND, LRU, RND = 0, 1, 2
BACKEND_STABLE, BACKEND_TCGEN05 = 0, 1
LOG_VICTIMS, LOG_RELOADS, LOG_GRADUATED = 0, 1, 2

POLICY_CODES = {"minpend": MINPEND, "lru": LRU, "rnd": RND}

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_vp = ctypes.c_void_p
P_i64 = ctypes.POINTER(ctypes.c_int64)


class LayerDesc(ctypes.Structure):
    _fields_ = [
        ("num_vertices", c_i64), ("dst_lo", c_i64), ("dst_hi", c_i64),
        ("model", c_i32), ("gin_epsilon", ctypes.c_float),
        ("embed_dim", c_i64), ("agg_dim", c_i64), ("slot_count", c_i64),
        ("evict_batch", c_i64), ("policy", c_i32), ("record_log", c_i32),
        ("rnd_state", ctypes.c_uint64 * 4), ("device", c_i32),
        ("force_exact", c_i32),
    ]


class LayerMetricsC(ctypes.Structure):
    _fields_ = [
        ("messages", c_i64), ("evictions", c_i64), ("reloads", c_i64),
        ("unique_reloads", c_i64), ("admissions", c_i64),
        ("graduations", c_i64), ("hot_peak", c_i64),
        ("hot_slot_count", c_i64), ("chunks", c_i64),
        ("span_count", c_i64), ("span_sum", c_i64), ("span_q_lo", c_i64),
        ("span_q_hi", c_i64), ("incomplete", c_i64),
        ("first_incomplete", c_i64 * 16), ("cold_bytes_read", c_i64),
        ("cold_bytes_written", c_i64), ("fast_path", c_i32), ("pad_", c_i32),
    ]


_LIB = None


def _declare(lib):
    def fn(name, res, *args):
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = list(args)

    fn("atlas_last_error", ctypes.c_char_p)
    fn("atlas_abi_version", ctypes.c_int)
    fn("atlas_kernel_launches", c_i64)
    fn("atlas_graph_create", ctypes.c_int, c_i32, c_i64, c_i64, c_vp, c_vp,
       c_vp, c_i64, c_i64, c_vp, ctypes.POINTER(c_vp))
    fn("atlas_graph_destroy", None, c_vp)
    fn("atlas_graph_update", ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_vp,
       c_vp, c_vp)
    fn("atlas_graph_csc", ctypes.c_int, c_vp, ctypes.POINTER(c_vp),
       ctypes.POINTER(c_vp), P_i64)
    fn("atlas_layer_create", ctypes.c_int, ctypes.POINTER(LayerDesc), c_vp,
       c_vp, ctypes.POINTER(c_vp))
    fn("atlas_layer_destroy", None, c_vp)
    fn("atlas_layer_reset", ctypes.c_int, c_vp, c_vp)
    fn("atlas_layer_bind_graph", ctypes.c_int, c_vp, c_vp, c_vp)
    fn("atlas_chunk_submit", ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_i32,
       c_vp, c_vp, c_i64, c_vp)
    fn("atlas_chunk_graduated", ctypes.c_int, c_vp, c_vp, c_vp, c_i64, P_i64,
       c_vp, c_i64, P_i64)
    fn("atlas_layer_run_resident", ctypes.c_int, c_vp, c_vp, c_vp, c_i32,
       c_i64, c_i64, c_vp, c_vp)
    fn("atlas_layer_run_streamed", ctypes.c_int, c_vp, c_vp, c_vp, c_i32,
       c_i64, c_i64, c_i64, c_vp)
    fn("atlas_layer_run_pieces", ctypes.c_int, c_vp, c_vp, c_vp, c_i32,
       c_i64, c_vp, c_i32, c_vp, c_i64, c_vp)
    fn("atlas_layer_run_blocked", ctypes.c_int, c_vp, c_vp, c_vp, c_i32,
       c_i64, c_i64, c_vp, c_i32, c_vp, c_vp, c_i64, c_i32, c_vp, c_i32,
       c_i64, c_vp, c_i64, c_vp)
    fn("atlas_layer_record_bytes", ctypes.c_int, c_vp, P_i64)
    fn("atlas_layer_accumulator", ctypes.c_int, c_vp, ctypes.POINTER(c_vp),
       P_i64)
    fn("atlas_transform", ctypes.c_int, c_i32, c_vp, c_i64, c_i64, c_i64,
       c_vp, c_vp, c_i64, c_i32, c_vp, c_i32, c_i64, c_vp, c_vp)
    fn("atlas_transform_typed", ctypes.c_int, c_i32, c_vp, c_i32, c_i64,
       c_i64, c_i64, c_vp, c_vp, c_i64, c_i32, c_vp, c_i32, c_i64, c_vp,
       c_vp)
    fn("atlas_transform_er", ctypes.c_int, c_i32, c_vp, c_i32, c_i64,
       c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_i32, c_i64, c_vp, c_i32,
       c_i32, c_i32, c_vp)
    fn("atlas_layer_run_gat", ctypes.c_int, c_vp, c_vp, c_vp, c_i32, c_i64,
       c_i32, c_i32, c_i32, c_i32, c_i32, c_vp, c_i32, c_i32, ctypes.c_float,
       c_vp, c_i32, c_i64, c_vp, c_i64, c_vp)
    fn("atlas_layer_run_fused", ctypes.c_int, c_vp, c_vp, c_vp, c_i64, c_i32,
       c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_vp, c_i32,
       c_i64, c_vp, c_vp, c_i64, c_i32, c_vp)
    fn("atlas_layer_finish", ctypes.c_int, c_vp,
       ctypes.POINTER(LayerMetricsC))
    fn("atlas_layer_chunk_stats", ctypes.c_int, c_vp, c_vp, c_vp, c_i64,
       P_i64)
    fn("atlas_layer_log", ctypes.c_int, c_vp, c_i32, c_vp, c_i64, P_i64)
    fn("atlas_layer_state", ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_vp)
    fn("atlas_layer_timing", ctypes.c_int, c_vp, c_vp, c_i32)
    fn("atlas_reorder", ctypes.c_int, c_i32, c_i64, c_i64, c_vp, c_vp, c_vp,
       c_vp, c_vp, c_vp, c_vp, c_vp, c_vp)
    fn("atlas_spill_read", ctypes.c_int, ctypes.POINTER(ctypes.c_char_p),
       c_i32, c_i32, c_i64, c_i64, c_vp, c_vp, c_i32, P_i64)
    fn("atlas_spill_read_device", ctypes.c_int,
       ctypes.POINTER(ctypes.c_char_p), c_i32, c_i32, c_i64, c_i64, c_vp,
       c_vp, c_i32, P_i64, ctypes.POINTER(c_i32))
    fn("atlas_gds_status", ctypes.c_char_p)
    fn("atlas_spill_write", ctypes.c_int, ctypes.c_char_p, c_vp, c_i32, c_i64,
       c_i64, c_i64, c_i64, c_i64, c_i32, P_i64)
    fn("atlas_spill_write_runs", ctypes.c_int, ctypes.c_char_p, c_vp, c_i32,
       c_i64, c_i64, c_vp, c_vp, c_i64, c_i32, P_i64)
    fn("atlas_gather_replay", ctypes.c_int, c_i64, c_i64, c_vp, c_vp, c_i64,
       c_i64, P_i64)


EXPORTED = [
    "atlas_last_error", "atlas_abi_version", "atlas_kernel_launches",
    "atlas_graph_create", "atlas_graph_destroy", "atlas_graph_csc",
    "atlas_graph_update",
    "atlas_layer_create", "atlas_layer_destroy", "atlas_layer_reset",
    "atlas_chunk_submit",
    "atlas_chunk_graduated", "atlas_layer_run_resident",
    "atlas_layer_run_streamed", "atlas_layer_run_pieces",
    "atlas_layer_accumulator", "atlas_transform", "atlas_layer_finish",
    "atlas_layer_chunk_stats", "atlas_layer_log", "atlas_layer_state",
    "atlas_layer_timing", "atlas_reorder", "atlas_transform_typed",
    "atlas_layer_run_gat", "atlas_layer_run_fused", "atlas_layer_bind_graph",
    "atlas_spill_read", "atlas_spill_write", "atlas_gather_replay",
    "atlas_spill_write_runs", "atlas_layer_run_blocked",
    "atlas_layer_record_bytes", "atlas_spill_read_device",
    "atlas_gds_status", "atlas_transform_er",
]


def load_library(path=LIB_PATH):
    """dlopen + declare prototypes; works without a GPU (no compute)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not Path(path).exists():
        raise DeviceError(
            f"{path} is missing: build it with __graft_entry__.build() "
            f"(nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(os.fspath(path))
    _declare(lib)
    _LIB = lib
    return lib


def lib():
    """The library, after checking a CUDA device is usable."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the engine runs only on B200 "
                          "(sm_100a); there is no CPU fallback")
    return load_library()


def check(code: int) -> None:
    if code != 0:
        msg = load_library().atlas_last_error().decode(errors="replace")
        raise_for_status(code, msg)


def ptr(x) -> int:
    """Raw address of a numpy array or torch tensor (0 for None)."""
    if x is None:
        return 0
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def kernel_launches() -> int:
    return int(load_library().atlas_kernel_launches())


def raise_incomplete(metrics: LayerMetricsC) -> None:
    ids = list(metrics.first_incomplete)[:min(16, metrics.incomplete)]
    raise IncompleteLayerError(ids, int(metrics.incomplete))

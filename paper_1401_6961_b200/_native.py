"""ctypes binding of libhxf.so (include/hxf.h).

The library is built in-tree by ``__graft_entry__.build()`` (csrc/Makefile).
There is no CPU fallback: if the library or a CUDA device is missing, every
call raises.
"""

from __future__ import annotations

import ctypes
import os

from .basis import InvalidArgumentError

HERE = os.path.dirname(os.path.abspath(__file__))
# HXF_LIB: alternative build of the same library (profiling variants; tools only)
LIB_PATH = os.environ.get("HXF_LIB") or os.path.join(HERE, "libhxf.so")

HXF_OK, HXF_EINVAL, HXF_ELOGIC, HXF_ECUDA, HXF_ENOMEM = 0, 1, 2, 3, 4
NCASES = 9

EXPORTED = ("hxf_last_error", "hxf_version", "hxf_system_create", "hxf_system_destroy",
            "hxf_system_info", "hxf_pairs_build", "hxf_pairs_build_ovlp", "hxf_pairs_destroy", "hxf_pairs_ties", "hxf_pairs_download",
            "hxf_pairs_download_q", "hxf_pairs_overlap", "hxf_density_build",
            "hxf_density_destroy", "hxf_density_download", "hxf_density_download_pmax", "hxf_exchange", "hxf_exchange_direct", "hxf_frontier",
            "hxf_last_timings", "hxf_symmetrize", "hxf_fp64_peak", "hxf_launch_count",
            "hxf_fixed_to_double", "hxf_scratch_release", "hxf_hilbert_order",
            "hxf_partition_build", "hxf_block_mask", "hxf_block_slots", "hxf_block_pack",
            "hxf_block_unpack", "hxf_span_mask", "hxf_span_pack", "hxf_span_unpack", "hxf_fixed_fold")


class LogicError(RuntimeError):
    """Internal traversal invariant violated (exchange_naive.py:24-25)."""


class Counters(ctypes.Structure):
    _fields_ = [("tasks_visited", ctypes.c_int64),
                ("tasks_culled_screening", ctypes.c_int64),
                ("tasks_culled_absent", ctypes.c_int64),
                ("leaf_contractions", ctypes.c_int64),
                ("eri_shell_quartets", ctypes.c_int64),
                ("quartets_culled_leaf", ctypes.c_int64),
                ("tasks_expanded", ctypes.c_int64),
                ("children_spawned", ctypes.c_int64),
                ("links_culled_screening", ctypes.c_int64),
                ("links_culled_absent", ctypes.c_int64),
                ("case_tasks", ctypes.c_int64 * NCASES),
                ("case_leaf_tasks", ctypes.c_int64 * NCASES),
                ("ties_task", ctypes.c_int64),
                ("ties_leaf", ctypes.c_int64),
                ("prim_quartets", ctypes.c_int64),
                ("class_quartets", ctypes.c_int64 * 16),
                ("class_prim_quartets", ctypes.c_int64 * 16),
                ("culled_bound_ledger", ctypes.c_double),
                ("screen_bytes", ctypes.c_int64)]


TIE_STAGES = ("task", "leaf", "overlap")


class TieRecord(ctypes.Structure):
    """hxf_tie_record: one culling comparison within 1e-12 relative of its threshold."""
    _fields_ = [("stage", ctypes.c_int32),
                ("level", ctypes.c_int32),
                ("slot", ctypes.c_int32),
                ("decision", ctypes.c_int32),
                ("id", ctypes.c_int32 * 4),
                ("bound", ctypes.c_double),
                ("threshold", ctypes.c_double),
                ("contribution", ctypes.c_double)]

    def to_dict(self):
        return {"stage": TIE_STAGES[self.stage], "level": int(self.level), "slot": int(self.slot),
                "decision": "kept" if self.decision else "culled", "ids": tuple(int(v) for v in self.id),
                "bound": float(self.bound), "threshold": float(self.threshold),
                "contribution": float(self.contribution)}


class ExchangeOpts(ctypes.Structure):
    _fields_ = [("tau_2e", ctypes.c_double),
                ("mode", ctypes.c_int),
                ("symmetry", ctypes.c_int),
                ("evaluate", ctypes.c_int),
                ("K_on_device", ctypes.c_int),
                ("symmetrize", ctypes.c_int),
                ("shard_level", ctypes.c_int),
                ("shard_begin", ctypes.c_int64),
                ("shard_end", ctypes.c_int64),
                ("quartet_log", ctypes.POINTER(ctypes.c_int32)),
                ("log_capacity", ctypes.c_int64),
                ("log_count", ctypes.POINTER(ctypes.c_int64)),
                ("digest", ctypes.POINTER(ctypes.c_uint64)),
                ("digest_mod", ctypes.c_int),
                ("digest_rem", ctypes.c_int),
                ("K_fixed", ctypes.c_int),
                ("K_scale", ctypes.POINTER(ctypes.c_int)),
                ("shard_stride", ctypes.c_int64),
                ("shard_mask", ctypes.POINTER(ctypes.c_uint8)),
                ("root_level", ctypes.c_int),
                ("root_index", ctypes.c_int),
                ("tie_log", ctypes.POINTER(TieRecord)),
                ("tie_capacity", ctypes.c_int64),
                ("tie_count", ctypes.POINTER(ctypes.c_int64)),
                ("count_screen_bytes", ctypes.c_int)]


_lib = None


def lib():
    """Load libhxf.so once; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"CUDA extension missing: {LIB_PATH} (run __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    P = ctypes.POINTER
    L.hxf_last_error.restype = ctypes.c_char_p
    L.hxf_version.restype = i32
    L.hxf_system_create.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp,
                                    vp, P(vp)]
    L.hxf_system_destroy.argtypes = [vp]
    L.hxf_system_destroy.restype = None
    L.hxf_system_info.argtypes = [vp, P(i64), P(i64)]
    L.hxf_pairs_build.argtypes = [vp, dbl, vp, P(vp)]
    L.hxf_pairs_build_ovlp.argtypes = [vp, dbl, vp, i32, vp, P(vp)]
    L.hxf_pairs_destroy.argtypes = [vp]
    L.hxf_pairs_destroy.restype = None
    L.hxf_pairs_ties.argtypes = [vp, P(TieRecord), i64, P(i64)]
    L.hxf_pairs_download.argtypes = [vp, i32, vp, vp, vp, vp]
    L.hxf_pairs_download_q.argtypes = [vp, vp]
    L.hxf_pairs_overlap.argtypes = [vp, vp]
    L.hxf_density_build.argtypes = [vp, vp, i32, dbl, vp, P(vp)]
    L.hxf_density_destroy.argtypes = [vp]
    L.hxf_density_destroy.restype = None
    L.hxf_density_download.argtypes = [vp, i32, vp]
    L.hxf_density_download_pmax.argtypes = [vp, vp]
    L.hxf_exchange.argtypes = [vp, vp, vp, P(ExchangeOpts), vp, P(Counters), vp]
    L.hxf_exchange_direct.argtypes = [vp, vp, P(ExchangeOpts), vp, P(Counters), vp]
    L.hxf_frontier.argtypes = [vp, vp, vp, dbl, i32, i32, i32, P(i64), vp, i64, vp]
    L.hxf_last_timings.argtypes = [vp, i32]
    L.hxf_symmetrize.argtypes = [vp, i32, dbl, vp]
    L.hxf_fp64_peak.argtypes = [P(dbl), vp]
    L.hxf_launch_count.argtypes = [P(i64)]
    L.hxf_fixed_to_double.argtypes = [vp, i64, i32, vp, vp]
    L.hxf_scratch_release.argtypes = [P(i64)]
    L.hxf_hilbert_order.argtypes = [vp, i64, i32, i32, vp, vp, vp]
    L.hxf_block_mask.argtypes = [vp, i32, i32, vp, vp]
    L.hxf_block_slots.argtypes = [vp, i64, vp, P(i64), vp]
    L.hxf_block_pack.argtypes = [vp, i32, i32, vp, vp, vp, vp]
    L.hxf_block_unpack.argtypes = [vp, i32, i32, vp, vp, vp, vp]
    L.hxf_span_mask.argtypes = [vp, i32, vp, vp, i32, vp, vp]
    L.hxf_span_pack.argtypes = [vp, i32, i32, vp, vp, i32, i32, i32, vp, vp, i64, vp, vp]
    L.hxf_span_unpack.argtypes = [vp, i32, i32, vp, vp, i32, i32, i32, vp, vp, i64, vp, vp]
    L.hxf_fixed_fold.argtypes = [vp, i32, vp]
    L.hxf_partition_build.argtypes = [vp, i64, i32, vp, vp, i64, vp, i32, P(i64), P(i32), vp]
    _lib = L
    return L


def check(rc):
    """Map an hxf status code to the reference's exception types."""
    if rc == HXF_OK:
        return
    msg = lib().hxf_last_error().decode(errors="replace")
    if rc == HXF_EINVAL:
        raise InvalidArgumentError(msg)
    if rc == HXF_ELOGIC:
        raise LogicError(msg)
    raise RuntimeError(f"libhxf error {rc}: {msg}")


def ptr(arr):
    """Raw pointer of a contiguous numpy array (or torch tensor)."""
    if hasattr(arr, "data_ptr"):
        return ctypes.c_void_p(arr.data_ptr())
    return arr.ctypes.data_as(ctypes.c_void_p)


def current_stream():
    """cudaStream_t of torch's current stream when torch is loaded, else NULL."""
    try:
        import torch
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    except Exception:  # pragma: no cover
        pass
    return ctypes.c_void_p(0)


def release_scratch() -> int:
    """Return the library's cached build scratch to the CUDA pool (syncs the device);
    the bytes released.  Builds cache their scratch so steady-state builds allocate
    nothing (include/hxf.h, hxf_scratch_release)."""
    n = ctypes.c_int64(0)
    check(lib().hxf_scratch_release(ctypes.byref(n)))
    return int(n.value)

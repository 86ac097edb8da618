"""ctypes binding of libgpic.so (include/gpic.h) and status -> exception map.

The product path has no CPU fallback: if the library or a CUDA device is
missing, every entry point raises instead of computing anything.
"""

from __future__ import annotations

import ctypes as C
import os
import pathlib

from . import errors

LIB_PATH = pathlib.Path(os.environ.get("GPIC_LIB") or  # experiments: an alternative build
                        pathlib.Path(__file__).resolve().parent / "libgpic.so")

GPIC_OK = 0
GPIC_E_INVALID = 1
GPIC_E_ZERO_DEGREE = 2
GPIC_E_NONFINITE = 3
GPIC_E_NONPOS_TAU = 4
GPIC_E_EMPTY = 5
GPIC_E_K_TOO_LARGE = 6
GPIC_E_ZERO_VECTOR = 7

KIND_RBF = 0
KIND_COSINE = 1
GPIC_E_CUDA = 16
GPIC_E_COMM = 17
GPIC_E_UNSUPPORTED = 18

AFFINITY_TC = 0
AFFINITY_SIMT = 1

STORAGE_DENSE = 0
STORAGE_PACKED = 1
STORAGE_NONE = 2
STORAGE_PACKED16 = 3


class Ctl(C.Structure):
    """Mirror of struct gpic_ctl (256 bytes)."""

    _fields_ = [
        ("iter", C.c_int32),
        ("stop", C.c_int32),
        ("converged", C.c_int32),
        ("status", C.c_int32),
        ("err_index", C.c_int64),
        ("err_index2", C.c_int64),
        ("err_value", C.c_double),
        ("eps", C.c_double),
        ("max_iter", C.c_int32),
        ("nranks", C.c_int32),
        ("delta_bits", C.c_uint64),
        ("arrive", C.c_uint32 * 4),
        ("tau", C.c_double),
        ("sync_epoch", C.c_uint64),
        ("tau_gen", C.c_uint32),
        ("bar_count", C.c_uint32),
        ("bar_gen", C.c_uint32),
        ("pad", C.c_uint8 * (256 - 108)),
    ]


assert C.sizeof(Ctl) == 256

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
F64 = C.c_double

# name -> (restype, argtypes); every symbol include/gpic.h declares.
SIGNATURES = {
    "gpic_version": (C.c_char_p, []),
    "gpic_last_error": (C.c_char_p, []),
    "gpic_workspace_bytes": (I64, [I64, I32, I32, I64, I32]),
    "gpic_affinity_pitch": (I64, [I64]),
    "gpic_feature_pitch": (I32, [I32]),
    "gpic_row_pad": (I64, [I64]),
    "gpic_operand_floats": (I64, [I64, I32]),
    "gpic_ctl_init": (C.c_int, [P, F64, I32, P]),
    "gpic_prepare_points": (C.c_int, [P, I64, I32, I32, P, P, P, P, P, P]),
    "gpic_engine_for": (I32, [I32, I32, C.c_double, C.c_double, I32, I32]),
    "gpic_last_detail": (C.c_int, [P, P, P]),
    "gpic_malloc": (C.c_int, [I64, P]),
    "gpic_free": (C.c_int, [P]),
    "gpic_cluster_host_workspace_bytes": (I64, [I64, I32, I32, I32, I32]),
    "gpic_affinity_rbf": (C.c_int, [P, P, P, I64, I32, I64, I64, F64, I32, P, I64, P, P, P, P]),
    "gpic_affinity_cosine": (C.c_int, [P, P, P, I64, I32, I64, I64, I32, P, I64, P, P, P, P]),
    "gpic_initial_vector": (C.c_int, [P, I64, P, P, P, P, P]),
    "gpic_power_iterate": (C.c_int, [P, I64, P, I64, P, P, F64, I32, P, P, P, P, P]),
    "gpic_kmeans1d": (C.c_int, [P, I64, I32, I64, P, I32, F64, P, P, P, P]),
    "gpic_kmeans_scratch_bytes": (I64, [I64, I32]),
    "gpic_reduce_sum": (C.c_int, [P, I64, P, P, P]),
    "gpic_scale": (C.c_int, [P, I64, F64, P, P, I64, P]),
    "gpic_matvec": (C.c_int, [P, I64, I64, I64, P, P, P, P]),
    "gpic_generate_blobs": (C.c_int, [P, P, I64, I32, I32, C.c_uint64, F64, F64, P, P, P]),
    "gpic_row_stats": (C.c_int, [P, I64, I64, I64, P, P, P, P]),
    "gpic_packed_tiles": (I64, [I64]),
    "gpic_vector_pitch": (I64, [I64]),
    "gpic_mf_ypart_doubles": (I64, [I64, I32, I64]),
    "gpic_mf_degrees": (C.c_int, [P, P, P, I64, I32, I64, I64, F64, I32, P, P, P, P]),
    "gpic_sym_matvec": (C.c_int, [P, I64, P, P, P, P, P, P]),
    "gpic_sym_matvec16": (C.c_int, [P, I64, P, P, P, P, P, P]),
    "gpic_sym_matvec_sparse": (C.c_int, [P, I32, I64, P, P, P, P, P, P, P, P]),
    "gpic_cluster_workspace_layout": (C.c_int, [I64, I32, I32, I32, I32, P]),
    "gpic_cluster_pruned_work": (C.c_int, [P, I64, I32, I32, I32, I32, P, P, P]),
    "gpic_mf_shard_scratch_bytes": (I64, [I64, I32]),
    "gpic_cluster_permutation": (C.c_int, [P, I64, I32, I32, I32, P, P, P]),
    "gpic_mf_shard_build": (C.c_int, [P, P, P, P, I64, I32, C.c_double, I32, I32, P, P, P]),
    "gpic_cluster_mf_pass": (C.c_int, [P, I64, I32, I32, I32, C.c_double, I32, I32, P, P, P]),
    "gpic_sym_partial_floats": (I64, [I64]),
    "gpic_packed_shard_range": (C.c_int, [I64, I32, I32, P, P]),
    "gpic_packed_shard_tiles": (I64, [I64, I64, I64]),
    "gpic_prune_scratch_bytes": (I64, [I64, I32]),
    "gpic_packed_shard_ranges_pruned": (C.c_int, [P, P, I64, I32, F64, I32, P, P, P]),
    "gpic_packed_shard_scratch_bytes": (I64, [I64, I64, I64]),
    "gpic_packed_shard_build": (C.c_int, [P, P, P, I64, I32, I64, I64, C.c_double, I32, P, P, P, P,
                                          P]),
    "gpic_cluster_workspace_bytes": (I64, [I64, I32, I32, I32, I32]),
    # (x, n, d, sigma, kind, k, eps, max_iter, first, uniforms, impl, storage, v0,
    #  labels, v, hist, iters, converged, work, work_bytes, stream[, phase_ms])
    "gpic_cluster": (C.c_int, [P, I64, I32, F64, I32, I32, F64, I32, I64, P, I32, I32, P, P, P,
                               P, P, P, P, I64, P]),
    "gpic_cluster_timed": (C.c_int, [P, I64, I32, F64, I32, I32, F64, I32, I64, P, I32, I32, P, P,
                                     P, P, P, P, P, I64, P, P]),
    "gpic_batch_workspace_bytes": (I64, [P, I32, I32, I32, I32]),
    "gpic_cluster_batch": (C.c_int, [P, P, I32, I32, F64, I32, I32, P, I32, P, P, P, P, P, P, P,
                                     I64, P]),
    "gpic_cluster_host": (C.c_int, [P, I64, I32, F64, I32, I32, F64, I32, I64, P, I32, I32, P, P,
                                    P, P, P, P, P, I64, P]),
    "gpic_ctl_read": (C.c_int, [P, P, P]),
    "gpic_launch_count": (I64, []),
    "gpic_comm_create": (C.c_int, [I32, I32, I64, P, P]),
    "gpic_comm_open": (C.c_int, [P, P]),
    "gpic_comm_create_virtual": (C.c_int, [I32, I64, P]),
    "gpic_comm_destroy": (C.c_int, [P]),
    "gpic_comm_gather_degrees": (C.c_int, [P, P, I32, P, P]),
    "gpic_comm_iterate": (C.c_int, [P, P, I32, F64, I32, P, P, P, P, P]),
}

IPC_HANDLE_BYTES = 64
MAX_RANKS = 8


class Shard(C.Structure):
    """Mirror of struct gpic_shard."""

    _fields_ = [("a", C.c_void_p), ("lda", C.c_int64), ("deg", C.c_void_p),
                ("row_lo", C.c_int64), ("rows", C.c_int64), ("storage", C.c_int32),
                ("d", C.c_int32), ("xhi", C.c_void_p), ("xlo", C.c_void_p), ("sqn", C.c_void_p),
                ("sigma", C.c_double), ("kind", C.c_int32), ("ypart", C.c_void_p),
                ("x", C.c_void_p)]

_lib = None


def lib():
    """Load libgpic.so once; raise loudly if it was never built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1604_02700_b200._build` "
                "(or __graft_entry__.build()); there is no CPU fallback"
            )
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().gpic_last_error()
    return msg.decode() if msg else ""


def raise_for(code: int, ctl: Ctl | None = None, d: int = 1) -> None:
    """Map a GPIC_E_* code (plus the control block's detail) onto errors.py."""
    if code == GPIC_OK:
        return
    msg = last_error()
    if code == GPIC_E_ZERO_DEGREE:
        raise errors.ZeroDegree(ctl.err_index if ctl is not None else -1)
    if code == GPIC_E_NONFINITE:
        idx = ctl.err_index if ctl is not None else 0
        raise errors.NonFiniteEntry(idx // max(d, 1), idx % max(d, 1))
    if code == GPIC_E_NONPOS_TAU:
        raise errors.NonPositiveTau(ctl.err_value if ctl is not None else float("nan"))
    if code == GPIC_E_ZERO_VECTOR:
        raise errors.ZeroVector(ctl.err_index if ctl is not None else -1)
    if code == GPIC_E_EMPTY:
        raise errors.EmptyDataSet()
    if code == GPIC_E_K_TOO_LARGE:
        raise errors.KTooLarge(-1, -1)
    if code == GPIC_E_INVALID:
        raise errors.InvalidSpec(msg)
    raise errors.DeviceError(f"libgpic error {code}: {msg}")


def check(code: int) -> None:
    """For calls whose only failures are host-side (no control block)."""
    raise_for(code)

"""ctypes binding of libgconn.so (include/gconn.h).

This is the only place the package touches the native library.  There is no
CPU fallback: if the library or a CUDA device is missing, every compute entry
point raises NativeError.  Device memory and streams come from PyTorch
(plumbing); the kernels are libgconn's.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import ConfigError, MalformedInputError, NativeError

LIB_PATH = Path(__file__).resolve().parent / "libgconn.so"
# A/B experiments only (profiles/ab_*.sh): an in-tree variant of the library
# built with different compile-time tunings
if os.environ.get("GC_LIB_VARIANT"):
    LIB_PATH = Path(__file__).resolve().parent / "_variants" / f"libgconn_{os.environ['GC_LIB_VARIANT']}.so"

GC_OK, GC_ERR_CONFIG, GC_ERR_MALFORMED, GC_ERR_CUDA, GC_ERR_OOM, GC_ERR_ARG = 0, 2, 3, 4, 5, 6

# enum values (gconn.h)
SAMPLE = {"none": 0, "kout": 1, "hb": 2, "bfs": 3, "ldd": 4}
FINISH = {"async": 0, "hooks": 1, "early": 2, "rem_lock": 3, "rem_cas": 4, "jtb": 5,
          "sv": 6, "lt": 7, "stergiou": 8, "lp": 9}
FIND = {"naive": 0, "split": 1, "halve": 2, "compress": 3, "twotry": 4}
SPLICE = {"none": 0, "split": 1, "halve": 2, "splice": 3}
LT_CONNECT = {"connect": 0, "parent_connect": 1, "extended_connect": 2}
LT_UPDATE = {"update": 0, "root_update": 1}
LT_SHORTCUT = {"shortcut": 0, "full_shortcut": 1}
KOUT_MODE = {"first_k": 0, "first_plus_random": 1}


class Csr(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("offsets", C.c_void_p), ("targets", C.c_void_p)]


class Spec(C.Structure):
    _fields_ = [("sample", C.c_int32), ("finish", C.c_int32), ("find", C.c_int32),
                ("splice", C.c_int32), ("lt_connect", C.c_int32), ("lt_update", C.c_int32),
                ("lt_shortcut", C.c_int32), ("lt_alter", C.c_int32), ("kout_k", C.c_int32),
                ("kout_mode", C.c_int32), ("hb_edges", C.c_int32), ("reserved0", C.c_int32),
                ("bfs_source", C.c_int64), ("seed", C.c_uint64), ("ldd_beta", C.c_double),
                ("jtb_ranks", C.c_void_p), ("kout_rand_offsets", C.c_void_p),
                ("bfs_probes", C.c_void_p), ("bfs_nprobes", C.c_int32), ("reserved1", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("t_sample_ms", C.c_double), ("t_finish_ms", C.c_double),
                ("t_finalize_ms", C.c_double), ("insp_sample", C.c_int64),
                ("insp_finish", C.c_int64), ("rounds", C.c_int64), ("components", C.c_int64),
                ("l_max", C.c_int64), ("lmax_count", C.c_int64), ("n_active", C.c_int64),
                ("ic_count", C.c_int64), ("t_sample_kernel_ms", C.c_double),
                ("t_finish_kernel_ms", C.c_double)]


_VP, _I64, _I32, _SZ = C.c_void_p, C.c_int64, C.c_int32, C.c_size_t
_SIGNATURES = {
    "gc_last_error": (C.c_char_p, []),
    "gc_version": (C.c_char_p, []),
    "gc_launch_count": (C.c_longlong, []),
    "gc_workspace_size": (_SZ, [_I64, _I64, C.POINTER(Spec)]),
    "gc_static_cc": (C.c_int, [C.POINTER(Csr), C.POINTER(Spec), _VP, _VP, C.c_int,
                               C.POINTER(Stats), _VP, _SZ, _VP]),
    "gc_plan_create": (C.c_int, [C.POINTER(Csr), C.POINTER(Spec), _VP, _VP, _SZ, _VP, C.POINTER(_VP)]),
    "gc_plan_run": (C.c_int, [_VP, C.POINTER(Stats)]),
    "gc_plan_destroy": (None, [_VP]),
    "gc_spanning_forest": (C.c_int, [C.POINTER(Csr), C.POINTER(Spec), _VP, _VP, _VP, C.POINTER(Stats),
                                     _VP, _SZ, _VP]),
    "gc_union_edges_list": (C.c_int, [_VP, _I64, _VP, _VP, _I64, C.POINTER(Spec), _VP, _VP, _VP, _VP, _VP]),
    "gc_incr_insert_list": (C.c_int, [_VP, _VP, _VP, _I64, _VP, _VP, _VP, C.POINTER(Stats)]),
    "gc_finish_phase": (C.c_int, [C.POINTER(Csr), C.POINTER(Spec), _VP, _I64, C.POINTER(Stats),
                                  _VP, _SZ, _VP]),
    "gc_label_finalization": (C.c_int, [_VP, _I64, _VP, _SZ, _VP]),
    "gc_union_edges": (C.c_int, [_VP, _I64, _VP, _VP, _I64, C.POINTER(Spec), _VP, _VP, _VP, _VP]),
    "gc_incr_create": (C.c_int, [_I64, C.POINTER(Spec), _VP, C.POINTER(_VP)]),
    "gc_incr_batch": (C.c_int, [_VP, _VP, _VP, _VP, _I64, _VP, C.c_int, C.POINTER(Stats)]),
    "gc_incr_insert": (C.c_int, [_VP, _VP, _VP, _I64, C.POINTER(Stats)]),
    "gc_incr_query": (C.c_int, [_VP, _VP, _VP, _I64, _VP, C.POINTER(Stats)]),
    "gc_incr_state": (C.c_int, [_VP, _VP]),
    "gc_incr_state_view": (C.c_int, [_VP, C.POINTER(_VP), C.POINTER(_I64)]),
    "gc_incr_set_stream": (C.c_int, [_VP, _VP]),
    "gc_incr_labels": (C.c_int, [_VP, _VP, C.POINTER(_I64)]),
    "gc_incr_capacity": (_I64, [_VP]),
    "gc_incr_reserve": (C.c_int, [_VP, _I64]),
    "gc_incr_insert_async": (C.c_int, [_VP, _VP, _VP, _I64, _VP]),
    "gc_incr_destroy": (None, [_VP]),
    "gc_gen_rmat": (C.c_int, [_I32, _I64, _VP, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                              _VP, _VP, _VP]),
    "gc_gen_uniform_pow2": (C.c_int, [_I32, _I64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                      _VP, _VP, _VP]),
    "gc_build_csr": (C.c_int, [_I64, _VP, _VP, _I64, _VP, _VP, C.POINTER(_I64), _VP, _SZ, _VP]),
    "gc_build_csr_workspace": (_SZ, [_I64, _I64]),
    "gc_mt19937_fill": (C.c_int, [_VP, C.c_int32, _VP, _I64]),
    "gc_shard_sample": (C.c_int, [C.POINTER(Csr), C.POINTER(Spec), _I64, _I64, _VP, _VP, _VP, _VP,
                                  C.POINTER(Stats), _VP, _SZ, _VP]),
    "gc_shard_finish": (C.c_int, [C.POINTER(Csr), C.POINTER(Spec), _I64, _I64, _VP, _VP, _VP, _VP,
                                  C.POINTER(Stats), _VP, _SZ, _VP]),
    "gc_shard_summary_workspace": (_SZ, [_I64]),
    "gc_shard_summary": (C.c_int, [_VP, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _SZ, _VP]),
    "gc_shard_absorb": (C.c_int, [_VP, _I64, _VP, _VP, C.c_int32, _VP, _VP, _SZ, _VP]),
    "gc_shard_join": (C.c_int, [_VP, _I64, _VP, _VP, C.c_int32, _VP, _VP, _I64, C.POINTER(Spec), _VP, _SZ, _VP]),
    "gc_dbfs_init": (C.c_int, [_I64, _I64, _VP, _VP, _VP, _VP]),
    "gc_dbfs_marks": (C.c_int, [C.POINTER(Csr), _I64, _I64, _VP, _VP, _VP, _VP, _VP, _VP]),
    "gc_dbfs_merge_marks": (C.c_int, [_I64, _VP, _I64, _VP, _VP, _VP]),
    "gc_dbfs_claim": (C.c_int, [C.POINTER(Csr), _I64, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "gc_dbfs_merge_claim": (C.c_int, [C.POINTER(Csr), _I64, _I64, _VP, _VP, _VP, _VP, _I64, _VP, _VP, _VP, _VP,
                                      _VP]),
    "gc_dbfs_advance": (C.c_int, [_I64, _VP, _VP, _VP, _VP, _VP]),
    "gc_dbfs_finish": (C.c_int, [C.POINTER(Csr), _I64, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _SZ,
                                 _VP]),
    "gc_comm_init": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(_VP)]),
    "gc_comm_destroy": (None, [_VP]),
    "gc_comm_size": (C.c_int, [_VP]),
    "gc_comm_is_loopback": (C.c_int, [_VP]),
    "gc_comm_static_cc": (C.c_int, [_VP, C.POINTER(Csr), C.POINTER(_I64), C.POINTER(_I64), C.POINTER(Spec),
                                    C.POINTER(_VP), C.POINTER(Stats)]),
    "gc_comm_spanning_forest": (C.c_int, [_VP, C.POINTER(Csr), C.POINTER(_I64), C.POINTER(_I64), C.POINTER(Spec),
                                          C.POINTER(_VP), C.POINTER(_VP), C.POINTER(_VP), C.POINTER(_I64),
                                          C.POINTER(Stats)]),
    "gc_check_csr": (C.c_int, [C.POINTER(Csr), _VP]),
    "gc_find_batch": (C.c_int, [_VP, _I64, _VP, _I64, C.c_int32, _VP, _VP]),
    "gc_canonical_labels": (C.c_int, [_VP, _I64, _VP, _SZ, _VP]),
    "gc_edges_exist": (C.c_int, [C.POINTER(Csr), _VP, _VP, _I64, _VP, _VP]),
    "gc_label_census": (C.c_int, [C.POINTER(Csr), _VP, _VP, C.POINTER(_I64), _VP, _SZ, _VP]),
}

_lock = threading.Lock()
_lib = None


def lib():
    """Load libgconn.so once; raise NativeError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                  "(there is no CPU fallback)")
            h = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_LOCAL", 0))
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def check(status: int) -> None:
    if status == GC_OK:
        return
    msg = (lib().gc_last_error() or b"").decode(errors="replace")
    if status == GC_ERR_CONFIG:
        raise ConfigError(msg)
    if status == GC_ERR_MALFORMED:
        raise MalformedInputError(msg)
    raise NativeError(f"libgconn status {status}: {msg}")


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)

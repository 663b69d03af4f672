"""ctypes binding of libbltc.so (include/bltc.h).

There is no CPU fallback: if the CUDA library is missing or fails to load,
every entry point raises.  The library is built in-tree by
``paper_2003_01836_b200.build_ext.build()`` (``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbltc.so")

BLTC_OK = 0
BLTC_ERR_VALUE = -1
BLTC_ERR_CUDA = -2
BLTC_ERR_STATE = -3
BLTC_ERR_UNSUPPORTED = -4
MODE_PARITY = 0
MODE_FAST = 1
MODE_STRICT = 2

_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_vp = ctypes.c_void_p


class Params(ctypes.Structure):
    _fields_ = [("theta", ctypes.c_double), ("degree", ctypes.c_int32),
                ("kernel_code", ctypes.c_int32), ("leaf_size", ctypes.c_int64),
                ("batch_size", ctypes.c_int64), ("kappa", ctypes.c_double),
                ("mode", ctypes.c_int32), ("all_moments", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("n_clusters", ctypes.c_int64), ("n_batches", ctypes.c_int64),
                ("direct_pairs", ctypes.c_int64), ("approx_pairs", ctypes.c_int64),
                ("setup_s", ctypes.c_double), ("precompute_s", ctypes.c_double),
                ("compute_s", ctypes.c_double), ("total_s", ctypes.c_double),
                ("h2d_s", ctypes.c_double), ("d2h_s", ctypes.c_double),
                ("far_s", ctypes.c_double), ("near_s", ctypes.c_double),
                ("n_moments", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("tree_depth", ctypes.c_int32), ("batch_depth", ctypes.c_int32),
                ("packed", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("n_recomputed", ctypes.c_int64), ("strict_s", ctypes.c_double)]


class Sizes(ctypes.Structure):
    _fields_ = [("n_sources", ctypes.c_int64), ("n_targets", ctypes.c_int64),
                ("n_clusters", ctypes.c_int64), ("n_batches", ctypes.c_int64),
                ("n_approx", ctypes.c_int64), ("n_direct", ctypes.c_int64),
                ("n_moments", ctypes.c_int64), ("degree", ctypes.c_int32),
                ("tree_depth", ctypes.c_int32), ("batch_depth", ctypes.c_int32),
                ("n_groups", ctypes.c_int32)]


class PublishSizes(ctypes.Structure):
    _fields_ = [("n_clusters", ctypes.c_int64), ("n_particles", ctypes.c_int64),
                ("n_moment_rows", ctypes.c_int64), ("record_doubles", ctypes.c_int64)]


# name -> (restype, argtypes); every symbol include/bltc.h declares.
SIGNATURES = {
    "bltc_last_error": (ctypes.c_char_p, []),
    "bltc_version": (ctypes.c_char_p, []),
    "bltc_create": (ctypes.c_int, [ctypes.c_int, _vp, ctypes.POINTER(_vp)]),
    "bltc_destroy": (ctypes.c_int, [_vp]),
    "bltc_set_timing": (ctypes.c_int, [_vp, ctypes.c_int]),
    "bltc_build": (ctypes.c_int, [_vp, ctypes.POINTER(Params), _f64p, ctypes.c_int64,
                                  _f64p, _f64p, _f64p, ctypes.c_int64, _f64p, _f64p, _f64p,
                                  _f64p, ctypes.c_int32, ctypes.POINTER(Stats)]),
    "bltc_treecode": (ctypes.c_int, [_vp, ctypes.POINTER(Params), _f64p, ctypes.c_int64,
                                     _f64p, _f64p, _f64p, ctypes.c_int64, _f64p, _f64p, _f64p,
                                     _f64p, ctypes.c_int32, _f64p, ctypes.POINTER(Stats)]),
    "bltc_treecode_device": (ctypes.c_int, [_vp, ctypes.POINTER(Params), _f64p, ctypes.c_int64,
                                            _vp, _vp, _vp, ctypes.c_int64, _vp, _vp, _vp, _vp,
                                            ctypes.c_int32, _vp, ctypes.POINTER(Stats)]),
    "bltc_get_sizes": (ctypes.c_int, [_vp, ctypes.POINTER(Sizes)]),
    "bltc_export_tree": (ctypes.c_int, [_vp, ctypes.c_int, _i64p, _i64p, _i64p, _i64p, _f64p,
                                        _f64p, _i64p, _i64p, _i32p]),
    "bltc_export_batches": (ctypes.c_int, [_vp, _i64p, _i64p, _f64p, _f64p]),
    "bltc_export_lists": (ctypes.c_int, [_vp, _i64p, _i64p, _i64p, _i64p]),
    "bltc_export_moments": (ctypes.c_int, [_vp, _i64p, _f64p]),
    "bltc_rank_build": (ctypes.c_int, [_vp, ctypes.POINTER(Params), _f64p, ctypes.c_int64, _vp,
                                       _vp, _vp, _vp, ctypes.c_int32]),
    "bltc_rank_set_domain": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_double),
                                            ctypes.POINTER(ctypes.c_double)]),
    "bltc_rank_set_domain_boxes": (ctypes.c_int, [_vp, ctypes.c_int64,
                                                  ctypes.POINTER(ctypes.c_double)]),
    "bltc_domain_cells": (ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double), ctypes.c_int32,
                                         ctypes.POINTER(ctypes.c_double), _i64p]),
    "bltc_rank_publish_sizes": (ctypes.c_int, [_vp, ctypes.POINTER(PublishSizes)]),
    "bltc_rank_publish": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "bltc_rank_evaluate": (ctypes.c_int, [_vp, ctypes.POINTER(Params), ctypes.c_int32,
                                          ctypes.c_int32, _i64p, _i64p, _i64p,
                                          ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                          ctypes.POINTER(_vp), _vp, ctypes.c_int32,
                                          ctypes.POINTER(Stats)]),
    "bltc_rank_needs": (ctypes.c_int, [_vp, ctypes.POINTER(Params), ctypes.c_int32,
                                       ctypes.c_int32, _i64p, ctypes.POINTER(_vp), _vp]),
    "bltc_probe_fp64": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, _f64p]),
    "bltc_launch_count": (ctypes.c_int, [_i64p]),
    "bltc_libm_exp_device": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, _f64p, _f64p]),
    "bltc_strict_keep_bounds": (ctypes.c_int, [_vp, ctypes.c_int32]),
    "bltc_export_strict_bounds": (ctypes.c_int, [_vp, _f64p, _f64p]),
    "bltc_run_distributed": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                            ctypes.c_int32, ctypes.POINTER(Params), _f64p,
                                            ctypes.c_int64, _f64p, _f64p, _f64p, _f64p, _i64p,
                                            _i64p, _f64p, ctypes.POINTER(Stats)]),
    "bltc_philox_uniform": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
                                           ctypes.POINTER(ctypes.c_uint64), ctypes.c_int64,
                                           ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                           ctypes.POINTER(_vp)]),
    "bltc_stage_lists": (ctypes.c_int, [_vp, ctypes.POINTER(Params), ctypes.c_int64, _i64p,
                                        _i64p, _f64p, _f64p, ctypes.c_int64, _i64p, _i64p,
                                        _f64p, _f64p, _i64p, _i64p, _i64p, _i64p]),
    "bltc_stage_moments": (ctypes.c_int, [_vp, ctypes.POINTER(Params), _f64p, ctypes.c_int64,
                                          _f64p, _f64p, _f64p, _f64p, ctypes.c_int64, _i64p,
                                          _i64p, _f64p, _f64p, ctypes.c_int64, _i64p, _f64p]),
    "bltc_stage_potentials": (ctypes.c_int, [_vp, ctypes.POINTER(Params), _f64p, ctypes.c_int64,
                                             _f64p, _f64p, _f64p, ctypes.c_int64, _i64p, _i64p,
                                             _f64p, _f64p, ctypes.c_int64, _f64p, _f64p, _f64p,
                                             _f64p, ctypes.c_int64, _i64p, _i64p, _f64p, _f64p,
                                             _i64p, _i64p, _i64p, _i64p, _i64p, ctypes.c_int64,
                                             _f64p, _i64p, _f64p, ctypes.POINTER(Stats)]),
    "bltc_direct_sum": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_double, ctypes.c_int32,
                                       ctypes.c_int64, _i64p, ctypes.c_int64, _f64p, _f64p,
                                       _f64p, ctypes.c_int64, _f64p, _f64p, _f64p, _f64p,
                                       _f64p]),
}

_lib = None


class BltcError(RuntimeError):
    """A CUDA-side failure inside libbltc."""


def load():
    """Load libbltc.so; raises if it is missing (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with paper_2003_01836_b200.build_ext.build() "
            "(the BLTC path has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == BLTC_OK:
        return
    msg = load().bltc_last_error().decode(errors="replace")
    if rc == BLTC_ERR_VALUE:
        raise ValueError(msg)
    if rc == BLTC_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == BLTC_ERR_STATE:
        raise RuntimeError(msg)
    raise BltcError(msg)


def f64p(a):
    return a.ctypes.data_as(_f64p)


def i64p(a):
    return a.ctypes.data_as(_i64p)


def i32p(a):
    return a.ctypes.data_as(_i32p)

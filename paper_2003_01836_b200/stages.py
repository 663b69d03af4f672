"""Stage-level drop-ins: each pipeline stage on structures the caller built.

The reference composes ``treecode_potentials`` from stages
(engine.py:350-372): ``build_interaction_lists`` (engine.py:128-130),
``compute_all_moments`` (moments.py:147-150) and ``compute_potentials``
(engine.py:315-335).  These functions run one stage on libbltc's CUDA
kernels (``bltc_stage_lists`` / ``bltc_stage_moments`` /
``bltc_stage_potentials``) on the caller's tree, batches, lists and moments,
so a stage can be swapped in alone -- and checked bit for bit in PARITY mode
against the reference's own upstream structures.

Inputs are the reference's objects (duck typed: ``SourceTree`` with
``clusters`` / ``points`` / ``charges``, ``BatchSet`` with ``batches`` /
``points`` / ``perm``, ``InteractionLists`` with ``approx`` / ``direct``,
``ClusterMoments`` with ``q_hat``) or flat arrays (``FlatTree``,
``FlatBatches``, ``FlatLists``), e.g. the oracle's or ``Context.export_*``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import RunStats, cheb_nodes, default_context, make_params


@dataclass(eq=False)
class FlatTree:
    """BFS cluster arrays (tree.py:198-217) + sources in cluster order."""

    start: np.ndarray
    stop: np.ndarray
    lo: np.ndarray            # [n][3]
    hi: np.ndarray
    child_start: np.ndarray
    child_count: np.ndarray
    x: np.ndarray | None = None
    y: np.ndarray | None = None
    z: np.ndarray | None = None
    q: np.ndarray | None = None


@dataclass(eq=False)
class FlatBatches:
    start: np.ndarray
    stop: np.ndarray
    center: np.ndarray        # [nb][3]
    radius: np.ndarray
    x: np.ndarray | None = None   # targets in batch order
    y: np.ndarray | None = None
    z: np.ndarray | None = None
    perm: np.ndarray | None = None   # original index -> batch-order position


@dataclass(eq=False)
class FlatLists:
    a_ptr: np.ndarray
    a_idx: np.ndarray
    d_ptr: np.ndarray
    d_idx: np.ndarray

    @property
    def approx(self) -> list:
        return [self.a_idx[self.a_ptr[b]:self.a_ptr[b + 1]].tolist()
                for b in range(len(self.a_ptr) - 1)]

    @property
    def direct(self) -> list:
        return [self.d_idx[self.d_ptr[b]:self.d_ptr[b + 1]].tolist()
                for b in range(len(self.d_ptr) - 1)]


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def flat_tree(tree) -> FlatTree:
    """A reference SourceTree (tree.py:191-222) or a flat tree."""
    if isinstance(tree, FlatTree):
        return tree
    if hasattr(tree, "clusters"):
        cl = tree.clusters
        t = FlatTree(start=_i64([c.start for c in cl]), stop=_i64([c.stop for c in cl]),
                     lo=_f64([c.box.lo for c in cl]).reshape(-1, 3),
                     hi=_f64([c.box.hi for c in cl]).reshape(-1, 3),
                     child_start=_i64([c.children[0].index if c.children else 0 for c in cl]),
                     child_count=_i64([len(c.children) for c in cl]))
        t.x, t.y, t.z = _f64(tree.points.x), _f64(tree.points.y), _f64(tree.points.z)
        t.q = _f64(tree.charges)
        return t
    # any object with the flat attribute names (e.g. the oracle's Tree)
    cs = _i64(tree.child_start)
    t = FlatTree(start=_i64(tree.start), stop=_i64(tree.stop), lo=_f64(tree.lo).reshape(-1, 3),
                 hi=_f64(tree.hi).reshape(-1, 3), child_start=np.where(cs < 0, 0, cs),
                 child_count=_i64(tree.child_count))
    for k in ("x", "y", "z", "q"):
        v = getattr(tree, k, None)
        setattr(t, k, None if v is None else _f64(v))
    return t


def flat_batches(batch_set) -> FlatBatches:
    """A reference BatchSet (tree.py:225-253) or flat batches."""
    if isinstance(batch_set, FlatBatches):
        return batch_set
    if hasattr(batch_set, "batches"):
        bs = batch_set.batches
        fb = FlatBatches(start=_i64([b.start for b in bs]), stop=_i64([b.stop for b in bs]),
                         center=_f64([b.center for b in bs]).reshape(-1, 3),
                         radius=_f64([b.radius for b in bs]))
        p = batch_set.points
        fb.x, fb.y, fb.z = _f64(p.x), _f64(p.y), _f64(p.z)
        fb.perm = _i64(batch_set.perm)
        return fb
    fb = FlatBatches(start=_i64(batch_set.start), stop=_i64(batch_set.stop),
                     center=_f64(batch_set.center).reshape(-1, 3), radius=_f64(batch_set.radius))
    for k in ("x", "y", "z", "perm"):
        v = getattr(batch_set, k, None)
        setattr(fb, k, None if v is None else (_i64(v) if k == "perm" else _f64(v)))
    return fb


def flat_lists(lists) -> FlatLists:
    """Reference InteractionLists (per-batch lists of cluster ids) or CSR."""
    if isinstance(lists, FlatLists):
        return lists
    if hasattr(lists, "a_ptr"):
        return FlatLists(_i64(lists.a_ptr), _i64(lists.a_idx), _i64(lists.d_ptr),
                         _i64(lists.d_idx))

    def csr(ll):
        ptr = np.zeros(len(ll) + 1, dtype=np.int64)
        ptr[1:] = np.cumsum([len(x) for x in ll])
        idx = _i64(np.concatenate([np.asarray(x, dtype=np.int64) for x in ll]) if ll else [])
        return ptr, idx
    a_ptr, a_idx = csr(lists.approx)
    d_ptr, d_idx = csr(lists.direct)
    return FlatLists(a_ptr, a_idx, d_ptr, d_idx)


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t)) if a is not None else None


def _f(a):
    return _p(a, ctypes.c_double)


def _l(a):
    return _p(a, ctypes.c_int64)


def build_interaction_lists(batch_set, tree, config, context=None) -> FlatLists:
    """engine.py:128-130 on the device, from the caller's batches and tree."""
    ctx = context or default_context()
    b, t = flat_batches(batch_set), flat_tree(tree)
    params = make_params(config, "parity")
    na, nd = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(ctx._lib.bltc_stage_lists(
        ctx.handle, ctypes.byref(params), len(b.start), _l(b.start), _l(b.stop),
        _f(_f64(b.center)), _f(b.radius), len(t.start), _l(t.start), _l(t.stop),
        _f(_f64(t.lo)), _f(_f64(t.hi)), _l(t.child_start), _l(t.child_count), ctypes.byref(na),
        ctypes.byref(nd)))
    nb = len(b.start)
    out = FlatLists(np.empty(nb + 1, np.int64), np.empty(max(1, na.value), np.int64),
                    np.empty(nb + 1, np.int64), np.empty(max(1, nd.value), np.int64))
    _lib.check(ctx._lib.bltc_export_lists(ctx.handle, _l(out.a_ptr), _l(out.a_idx),
                                          _l(out.d_ptr), _l(out.d_idx)))
    out.a_idx, out.d_idx = out.a_idx[:na.value], out.d_idx[:nd.value]
    return out


def compute_moments(tree, config, cluster_ids=None, mode=None, context=None) -> np.ndarray:
    """compute_modified_charges (moments.py:132-144) of ``cluster_ids`` (all
    eligible clusters if None, as compute_all_moments, moments.py:147-150):
    rows [len(ids)][(n+1)^3]."""
    ctx = context or default_context()
    t = flat_tree(tree)
    if t.x is None or t.q is None:
        raise ValueError("the tree needs its sources (x, y, z, q in cluster order)")
    if cluster_ids is None:
        ext = _f64(t.hi) - _f64(t.lo)
        cluster_ids = np.nonzero(np.all(ext >= 1e-14, axis=1))[0]   # tree.py:205-206
    ids = _i64(cluster_ids)
    params = make_params(config, mode)
    m3 = (params.degree + 1) ** 3
    rows = np.empty((len(ids), m3))
    nodes = cheb_nodes(params.degree)
    _lib.check(ctx._lib.bltc_stage_moments(
        ctx.handle, ctypes.byref(params), _f(nodes), len(t.x), _f(t.x), _f(t.y), _f(t.z),
        _f(t.q), len(t.start), _l(t.start), _l(t.stop), _f(_f64(t.lo)), _f(_f64(t.hi)),
        len(ids), _l(ids), _f(rows)))
    return rows


@dataclass(eq=False)
class ClusterMoments:
    """moments.py:40-43: one cluster's modified charges, k1-major."""

    cluster_index: int
    q_hat: np.ndarray


def compute_all_moments(tree, config, mode=None, context=None) -> list:
    """compute_all_moments (moments.py:147-150) on the device: a list indexed
    by cluster, ClusterMoments for every eligible cluster (all extents
    >= 1e-14, tree.py:205-206), None otherwise."""
    t = flat_tree(tree)
    ext = _f64(t.hi) - _f64(t.lo)
    ids = np.nonzero(np.all(ext >= 1e-14, axis=1))[0]
    rows = compute_moments(tree, config, ids, mode=mode, context=context)
    out = [None] * len(t.start)
    for k, ci in enumerate(ids):
        out[int(ci)] = ClusterMoments(int(ci), rows[k])
    return out


def compute_potentials(batch_set, tree, moments, lists, config, threads: int = 1,
                       mode=None, moment_row=None, context=None, return_stats: bool = False):
    """engine.py:315-335 on the device: all approximations then all direct
    sums per batch; phi in the original target order when the batches carry
    ``perm`` (batch order otherwise).  ``moments``: the reference's list of
    ClusterMoments-or-None indexed by cluster, or rows [n_rows][(n+1)^3] with
    ``moment_row`` (cluster -> row, -1 for none).  Returns phi, like the
    reference; (phi, RunStats) with ``return_stats``."""
    del threads
    ctx = context or default_context()
    b, t, L = flat_batches(batch_set), flat_tree(tree), flat_lists(lists)
    if b.x is None or t.x is None or t.q is None:
        raise ValueError("batches need their targets and the tree its sources")
    params = make_params(config, mode)
    m3 = (params.degree + 1) ** 3
    nc = len(t.start)
    if moment_row is None:
        mrow = np.full(nc, -1, dtype=np.int64)
        rows = []
        for ci, mm in enumerate(moments):
            if mm is not None:
                mrow[ci] = len(rows)
                rows.append(np.asarray(getattr(mm, "q_hat", mm), dtype=np.float64))
        rows = _f64(np.stack(rows)) if rows else np.zeros((0, m3))
    else:
        mrow, rows = _i64(moment_row), _f64(moments).reshape(-1, m3)
    phi = np.empty(len(b.x))
    st = _lib.Stats()
    nodes = cheb_nodes(params.degree)
    _lib.check(ctx._lib.bltc_stage_potentials(
        ctx.handle, ctypes.byref(params), _f(nodes), len(b.x), _f(b.x), _f(b.y), _f(b.z),
        len(b.start), _l(b.start), _l(b.stop), _f(_f64(b.center)), _f(b.radius), len(t.x),
        _f(t.x), _f(t.y), _f(t.z), _f(t.q), nc, _l(t.start), _l(t.stop), _f(_f64(t.lo)),
        _f(_f64(t.hi)), _l(L.a_ptr), _l(L.a_idx) if len(L.a_idx) else None, _l(L.d_ptr),
        _l(L.d_idx) if len(L.d_idx) else None, _l(mrow), rows.shape[0],
        _f(rows) if rows.shape[0] else None, _l(b.perm), _f(phi), ctypes.byref(st)))
    return (phi, RunStats.from_c(st)) if return_stats else phi

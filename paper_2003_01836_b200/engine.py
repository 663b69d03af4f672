"""Drop-in BLTC evaluation entry point on B200 (engine.py of the reference).

``treecode_potentials(system, config, threads=1)`` keeps the reference's
signature and return value (engine.py:350-372): potentials in the caller's
original target order plus a :class:`RunStats`.  Every stage -- source tree,
target batches, interaction lists, moments, far/near-field sums,
un-permute -- runs in libbltc's sm_100a CUDA kernels; this module only
validates arguments (raising the reference's ``ValueError``s) and moves
buffers across the C ABI.

``system`` may be this package's :class:`~.particles.ParticleSystem` or the
reference's own object (duck typed: ``targets``/``sources`` with float64
``x, y, z``; ``charges``; ``targets is sources`` means coincident).
``config`` may be this package's :class:`EvalConfig` or the reference's.

Modes: ``"strict"`` (the default) runs the performance kernels on the
reference's own moments and certifies every target: a target whose FAST
value cannot be shown to lie within 0.5e-10 (relative) of the reference's is
recomputed in the reference's arithmetic, so every potential meets the
north-star 1e-10 per-target tolerance (``RunStats.n_recomputed`` counts the
recomputed ones).  ``"parity"`` reproduces the reference bit for bit for
every target (IEEE sqrt/div, no FMA, reference accumulation order);
``"fast"`` is the uncertified performance path (rsqrt + FMA, register-blocked
tiles, FMA-fused moments), within ~1e-13 of max|phi| of the reference.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .kernels import KernelSpec, coulomb
from .particles import ParticleSystem

DEFAULT_MODE = os.environ.get("BLTC_MODE", "strict")
_MODES = {"parity": _lib.MODE_PARITY, "fast": _lib.MODE_FAST, "strict": _lib.MODE_STRICT}


@dataclass(frozen=True)
class EvalConfig:
    """Treecode parameters for one run (engine.py:46-62)."""

    theta: float
    degree: int
    leaf_size: int = 2000
    batch_size: int = 2000
    kernel: KernelSpec = field(default_factory=coulomb)

    def __post_init__(self):
        if not (0.0 < self.theta <= 1.0):
            raise ValueError(f"theta must be in (0, 1], got {self.theta}")
        if self.degree < 0:
            raise ValueError("degree must be >= 0")
        if self.leaf_size < 1 or self.batch_size < 1:
            raise ValueError("leaf_size and batch_size must be >= 1")


@dataclass(eq=False)
class RunStats:
    """engine.py:338-347 plus device detail (times are CUDA-event seconds)."""

    n_clusters: int
    n_batches: int
    direct_pairs: int
    approx_pairs: int
    setup_s: float
    precompute_s: float
    compute_s: float
    total_s: float
    h2d_s: float = 0.0
    d2h_s: float = 0.0
    far_s: float = 0.0
    near_s: float = 0.0
    n_moments: int = 0
    kernel_launches: int = 0
    tree_depth: int = 0
    batch_depth: int = 0
    packed: int = 0
    n_recomputed: int = 0
    strict_s: float = 0.0

    @classmethod
    def from_c(cls, s: _lib.Stats) -> "RunStats":
        return cls(**{name: getattr(s, name) for name, _ in _lib.Stats._fields_
                      if name != "reserved"})


def cheb_nodes(degree: int) -> np.ndarray:
    """Normalised second-kind Chebyshev nodes s_k = sin(pi (n - 2k) / (2n))
    (interp.py:52), computed with numpy on the host so the device grids are
    bitwise those of the reference (no device sin)."""
    if degree == 0:
        return np.zeros(1)
    k = np.arange(degree + 1)
    return np.ascontiguousarray(np.sin(np.pi * (degree - 2 * k) / (2 * degree)))


def make_params(config, mode: str | None = None, all_moments: bool = False) -> _lib.Params:
    mode = DEFAULT_MODE if mode is None else mode
    if mode not in _MODES:
        raise ValueError(f"mode must be one of {sorted(_MODES)}, got {mode!r}")
    theta, degree = float(config.theta), int(config.degree)
    if not (0.0 < theta <= 1.0):
        raise ValueError(f"theta must be in (0, 1], got {theta}")
    if degree < 0:
        raise ValueError("degree must be >= 0")
    if int(config.leaf_size) < 1 or int(config.batch_size) < 1:
        raise ValueError("leaf_size and batch_size must be >= 1")
    kernel = config.kernel
    kappa = float(kernel.kappa)
    if not np.isfinite(kappa) or kappa < 0.0:
        raise ValueError(f"kappa must be finite and >= 0, got {kappa}")
    return _lib.Params(theta=theta, degree=degree, kernel_code=int(kernel.code),
                       leaf_size=int(config.leaf_size), batch_size=int(config.batch_size),
                       kappa=kappa, mode=_MODES[mode], all_moments=1 if all_moments else 0)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Context:
    """One libbltc context (device buffers + stream) on one CUDA device."""

    def __init__(self, device: int = -1, stream: int | None = None):
        """``stream``: None -- libbltc creates its own (non-blocking) stream;
        otherwise a CUDA stream handle, e.g. torch.cuda.current_stream().
        cuda_stream, whose value 0 means the legacy default stream (passed to
        libbltc as cudaStreamLegacy, so it really runs on that stream)."""
        self._lib = _lib.load()
        h = ctypes.c_void_p()
        handle = 0 if stream is None else (int(stream) or 1)   # 1 = cudaStreamLegacy
        _lib.check(self._lib.bltc_create(int(device), ctypes.c_void_p(handle), ctypes.byref(h)))
        self.handle = h
        # the torch-visible handle of the stream libbltc runs on (None: its own)
        self.stream = None if stream is None else int(stream)

    def close(self):
        if getattr(self, "handle", None):
            _lib.check(self._lib.bltc_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_timing(self, enable: bool) -> None:
        _lib.check(self._lib.bltc_set_timing(self.handle, 1 if enable else 0))

    # -- full pipeline -------------------------------------------------------
    def treecode(self, system, config, mode: str | None = None, all_moments: bool = False,
                 out: np.ndarray | None = None):
        p = make_params(config, mode, all_moments)
        t, s = system.targets, system.sources
        coincident = t is s
        sx, sy, sz = _f64(s.x), _f64(s.y), _f64(s.z)
        q = _f64(system.charges)
        if q.shape[0] != sx.shape[0]:
            raise ValueError("one charge per source particle required")
        if coincident:
            tx, ty, tz = sx, sy, sz
        else:
            tx, ty, tz = _f64(t.x), _f64(t.y), _f64(t.z)
        n_t, n_s = tx.shape[0], sx.shape[0]
        if n_s == 0 or n_t == 0:
            raise ValueError("cannot partition an empty particle set")
        phi = np.empty(n_t) if out is None else out
        st = _lib.Stats()
        nodes = cheb_nodes(p.degree)
        _lib.check(self._lib.bltc_treecode(
            self.handle, ctypes.byref(p), _lib.f64p(nodes), n_t, _lib.f64p(tx), _lib.f64p(ty),
            _lib.f64p(tz), n_s, _lib.f64p(sx), _lib.f64p(sy), _lib.f64p(sz), _lib.f64p(q),
            1 if coincident else 0, _lib.f64p(phi), ctypes.byref(st)))
        return phi, RunStats.from_c(st)

    def build(self, system, config, mode: str | None = None, all_moments: bool = True
              ) -> RunStats:
        """Tree, batches, lists and moments only (no evaluation): the setup and
        precompute phases of treecode_potentials (engine.py:353-362); read the
        structures with export_tree / export_batches / export_lists /
        export_moments."""
        p = make_params(config, mode, all_moments)
        t, s = system.targets, system.sources
        coincident = t is s
        sx, sy, sz = _f64(s.x), _f64(s.y), _f64(s.z)
        q = _f64(system.charges)
        if q.shape[0] != sx.shape[0]:
            raise ValueError("one charge per source particle required")
        tx, ty, tz = (sx, sy, sz) if coincident else (_f64(t.x), _f64(t.y), _f64(t.z))
        if sx.shape[0] == 0 or tx.shape[0] == 0:
            raise ValueError("cannot partition an empty particle set")
        st = _lib.Stats()
        _lib.check(self._lib.bltc_build(
            self.handle, ctypes.byref(p), _lib.f64p(cheb_nodes(p.degree)), tx.shape[0],
            _lib.f64p(tx), _lib.f64p(ty), _lib.f64p(tz), sx.shape[0], _lib.f64p(sx),
            _lib.f64p(sy), _lib.f64p(sz), _lib.f64p(q), 1 if coincident else 0,
            ctypes.byref(st)))
        return RunStats.from_c(st)

    def treecode_device(self, params: _lib.Params, n_t, tx, ty, tz, n_s, sx, sy, sz, q,
                        coincident: bool, phi_ptr) -> RunStats:
        """Device-pointer variant (inputs resident in HBM): raw integer pointers."""
        st = _lib.Stats()
        nodes = cheb_nodes(params.degree)
        _lib.check(self._lib.bltc_treecode_device(
            self.handle, ctypes.byref(params), _lib.f64p(nodes), int(n_t), tx, ty, tz, int(n_s),
            sx, sy, sz, q, 1 if coincident else 0, phi_ptr, ctypes.byref(st)))
        return RunStats.from_c(st)

    def direct_sum(self, system, kernel, sample=None, mode: str = "parity") -> np.ndarray:
        """Brute-force potentials at ``sample`` (all targets if None) on the
        device -- the reference harness's verification oracle (cli.py:130-149)."""
        t, s = system.targets, system.sources
        tx, ty, tz = _f64(t.x), _f64(t.y), _f64(t.z)
        sx, sy, sz, q = _f64(s.x), _f64(s.y), _f64(s.z), _f64(system.charges)
        idx = None if sample is None else np.ascontiguousarray(sample, dtype=np.int64)
        m = tx.shape[0] if idx is None else idx.shape[0]
        out = np.empty(m)
        _lib.check(self._lib.bltc_direct_sum(
            self.handle, int(kernel.code), float(kernel.kappa), _MODES[mode], m,
            None if idx is None else _lib.i64p(idx), tx.shape[0], _lib.f64p(tx), _lib.f64p(ty),
            _lib.f64p(tz), sx.shape[0], _lib.f64p(sx), _lib.f64p(sy), _lib.f64p(sz),
            _lib.f64p(q), _lib.f64p(out)))
        return out

    # -- distributed rank entry points (decomp.py:483-593) -----------------------
    def rank_build(self, params: _lib.Params, n: int, x, y, z, q, device_ptrs: bool) -> None:
        """Local tree, batches and moments of one rank.  x, y, z, q: numpy arrays
        (device_ptrs False) or raw device pointers (True)."""
        nodes = cheb_nodes(params.degree)
        if device_ptrs:
            args = [ctypes.c_void_p(int(v)) for v in (x, y, z, q)]
        else:
            args = [_lib.f64p(_f64(v)) for v in (x, y, z, q)]
            self._keep = (x, y, z, q)
        _lib.check(self._lib.bltc_rank_build(self.handle, ctypes.byref(params),
                                             _lib.f64p(nodes), int(n), *args,
                                             1 if device_ptrs else 0))

    def rank_set_domain(self, lo, hi) -> None:
        """The global target domain for the next rank_build (None: unset)."""
        if lo is None:
            _lib.check(self._lib.bltc_rank_set_domain(self.handle, None, None))
            return
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        hi = np.ascontiguousarray(hi, dtype=np.float64)
        _lib.check(self._lib.bltc_rank_set_domain(self.handle, _lib.f64p(lo), _lib.f64p(hi)))

    def rank_set_domain_boxes(self, boxes) -> None:
        """The global target domain as a union of boxes ([k, 6]: lo xyz, hi
        xyz; empty: unset) for the next rank_build."""
        b = np.ascontiguousarray(boxes, dtype=np.float64).reshape(-1, 6)
        _lib.check(self._lib.bltc_rank_set_domain_boxes(self.handle, b.shape[0], _lib.f64p(b)))

    def rank_publish_sizes(self) -> dict:
        ps = _lib.PublishSizes()
        _lib.check(self._lib.bltc_rank_publish_sizes(self.handle, ctypes.byref(ps)))
        return {name: getattr(ps, name) for name, _ in _lib.PublishSizes._fields_}

    def rank_publish(self, records_ptr: int, particles_ptr: int, moments_ptr: int) -> None:
        _lib.check(self._lib.bltc_rank_publish(self.handle, ctypes.c_void_p(records_ptr),
                                               ctypes.c_void_p(particles_ptr),
                                               ctypes.c_void_p(moments_ptr)))

    def rank_evaluate(self, params: _lib.Params, ranks: int, my_rank: int, n_clusters,
                      n_particles, n_moment_rows, records, particles, moments, phi_out,
                      device_ptrs: bool) -> RunStats:
        """Evaluate this rank's batches against the gathered forest (device
        pointers per owner rank, owner order 0..R-1)."""
        R = int(ranks)
        nc = np.ascontiguousarray(n_clusters, dtype=np.int64)
        npart = np.ascontiguousarray(n_particles, dtype=np.int64)
        nrow = np.ascontiguousarray(n_moment_rows, dtype=np.int64)
        arr = ctypes.c_void_p * R
        rec = arr(*[ctypes.c_void_p(int(v)) for v in records])
        par = arr(*[ctypes.c_void_p(int(v)) for v in particles])
        mom = arr(*[ctypes.c_void_p(int(v)) for v in moments])
        st = _lib.Stats()
        out = ctypes.c_void_p(int(phi_out)) if device_ptrs else \
            ctypes.c_void_p(phi_out.ctypes.data)
        _lib.check(self._lib.bltc_rank_evaluate(
            self.handle, ctypes.byref(params), R, int(my_rank), _lib.i64p(nc), _lib.i64p(npart),
            _lib.i64p(nrow), rec, par, mom, out, 1 if device_ptrs else 0, ctypes.byref(st)))
        return RunStats.from_c(st)

    def rank_needs(self, params: _lib.Params, ranks: int, my_rank: int, n_clusters, records,
                   flags_out_ptr: int) -> None:
        """LET step one: per cluster of every owner's tree (owner order
        0..R-1, device pointers), bit 0 = moment row needed, bit 1 =
        particles needed, written as int32 to the device buffer flags_out."""
        R = int(ranks)
        nc = np.ascontiguousarray(n_clusters, dtype=np.int64)
        rec = (ctypes.c_void_p * R)(*[ctypes.c_void_p(int(v)) for v in records])
        _lib.check(self._lib.bltc_rank_needs(self.handle, ctypes.byref(params), R, int(my_rank),
                                             _lib.i64p(nc), rec, ctypes.c_void_p(flags_out_ptr)))

    # -- stage exports of the last run (bit-exact structure checks) ------------
    def sizes(self) -> _lib.Sizes:
        sz = _lib.Sizes()
        _lib.check(self._lib.bltc_get_sizes(self.handle, ctypes.byref(sz)))
        return sz

    def export_tree(self, which: int = 0) -> dict:
        sz = self.sizes()
        n = sz.n_sources if which == 0 else sz.n_targets
        nn = ctypes.c_int64()
        _lib.check(self._lib.bltc_export_tree(self.handle, which, ctypes.byref(nn), None, None,
                                              None, None, None, None, None, None))
        nn = nn.value
        out = dict(perm=np.empty(n, np.int64), start=np.empty(nn, np.int64),
                   stop=np.empty(nn, np.int64), lo=np.empty((nn, 3)), hi=np.empty((nn, 3)),
                   child_start=np.empty(nn, np.int64), child_count=np.empty(nn, np.int64),
                   level=np.empty(nn, np.int32))
        _lib.check(self._lib.bltc_export_tree(
            self.handle, which, None, _lib.i64p(out["perm"]), _lib.i64p(out["start"]),
            _lib.i64p(out["stop"]), _lib.f64p(out["lo"]), _lib.f64p(out["hi"]),
            _lib.i64p(out["child_start"]), _lib.i64p(out["child_count"]),
            _lib.i32p(out["level"])))
        return out

    def export_batches(self) -> dict:
        nb = self.sizes().n_batches
        out = dict(start=np.empty(nb, np.int64), stop=np.empty(nb, np.int64),
                   center=np.empty((nb, 3)), radius=np.empty(nb))
        _lib.check(self._lib.bltc_export_batches(self.handle, _lib.i64p(out["start"]),
                                                 _lib.i64p(out["stop"]),
                                                 _lib.f64p(out["center"]),
                                                 _lib.f64p(out["radius"])))
        return out

    def export_lists(self) -> dict:
        sz = self.sizes()
        nseg = sz.n_batches * max(1, sz.n_groups)
        out = dict(a_ptr=np.empty(nseg + 1, np.int64), a_idx=np.empty(sz.n_approx, np.int64),
                   d_ptr=np.empty(nseg + 1, np.int64), d_idx=np.empty(sz.n_direct, np.int64))
        _lib.check(self._lib.bltc_export_lists(self.handle, _lib.i64p(out["a_ptr"]),
                                               _lib.i64p(out["a_idx"]), _lib.i64p(out["d_ptr"]),
                                               _lib.i64p(out["d_idx"])))
        return out

    def keep_strict_bounds(self, enable: bool = True) -> None:
        """Keep the STRICT certificate's per-target bound of the next runs."""
        _lib.check(self._lib.bltc_strict_keep_bounds(self.handle, 1 if enable else 0))

    def export_strict_bounds(self) -> tuple[np.ndarray, float]:
        """(S, Kc) of the last STRICT run: S_i = absum_i + farbound_i per target
        in the original order; a target is certified when Kc eps S_i <= 0.5e-10
        |phi_i| and recomputed in the reference's arithmetic otherwise."""
        n = self.sizes().n_targets
        out = np.empty(n)
        kc = ctypes.c_double()
        _lib.check(self._lib.bltc_export_strict_bounds(self.handle, _lib.f64p(out),
                                                       ctypes.byref(kc)))
        return out, kc.value

    def export_moments(self):
        sz = self.sizes()
        m3 = (sz.degree + 1) ** 3
        ids = np.empty(sz.n_moments, np.int64)
        rows = np.empty((sz.n_moments, m3))
        _lib.check(self._lib.bltc_export_moments(self.handle, _lib.i64p(ids), _lib.f64p(rows)))
        return ids, rows


_default_ctx: dict[int, Context] = {}


def default_context(device: int = -1) -> Context:
    ctx = _default_ctx.get(device)
    if ctx is None:
        ctx = Context(device)
        _default_ctx[device] = ctx
    return ctx


def treecode_potentials(system: ParticleSystem, config: EvalConfig, threads: int = 1,
                        mode: str | None = None, context: Context | None = None
                        ) -> tuple[np.ndarray, RunStats]:
    """Full pipeline on the GPU (engine.py:350-372).

    ``threads`` is accepted for signature compatibility and ignored: the
    device schedules target batches itself (the reference's results are
    thread-count invariant, test_engine.py:241-248, and so are these).
    """
    del threads
    ctx = context or default_context()
    return ctx.treecode(system, config, mode=mode)

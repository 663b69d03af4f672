"""Multi-rank BLTC evaluation: one rank per GPU (decomp.py of the reference).

``run_distributed(system, config, ranks, threads=1)`` keeps the reference's
signature and results (decomp.py:483-593): targets are partitioned by
recursive coordinate bisection (decomp.py:76-130, restated here on the host
with the same numpy order statistics so every rank's particle order -- and
therefore every bit of its tree -- matches the reference); each rank builds
its own source tree, target batches and moments on its GPU; the forest is
replicated by ONE all-gather of the published records (NCCL over NVLink when
``torch.distributed`` runs one process per GPU); each rank then evaluates
its batches against the local tree first and the remote trees in ascending
owner order (decomp.py:437-454), exactly the reference's accumulation order.

Exchange (``exchange=``):
* ``"let"`` (default) -- the reference's two-step locally essential tree
  (decomp.py:354-399, build_let) as collectives: (1) all-gather of every
  rank's tree records; each rank builds its batches' interaction lists
  against every remote tree on its GPU (``bltc_rank_needs``) and marks the
  clusters it approximates (moment rows needed) or sums directly (particle
  slices needed); (2) one all-to-all of the requested cluster ids and one
  all-to-all of exactly those moment rows and particle slices.  Nothing else
  moves, so the fetch statistics are the reference's (``let_violations``
  counts stay zero) and the evaluation sees the same data as the reference.
* ``"replicate"`` -- north_star's exchange and the default of the
  one-process-per-GPU runner (``DeviceRankRunner``, bench.py N > 1): one
  all-gather of three sizes per rank, then ONE all-gather of every rank's
  packed [tree records | particles | moment rows] block, published by
  libbltc straight into the send buffer (``publish_packed``).  Every rank
  holds a superset of its LET; on one NVSwitch box moving the whole forest
  (≈ 300 MB at 8M particles) costs well under a millisecond, less than the
  LET's extra plan / serve round trips.

Execution models:
* ``torch.distributed`` initialised with world_size == ranks: this process is
  one rank (its GPU = ``torch.cuda.current_device()``); the exchange is
  ``all_gather`` over the process group (NCCL).
* otherwise: the ranks run back to back in this process on one GPU and the
  exchange is a no-op (the published device buffers are read in place).

The per-rank device work goes through a rank engine; the product engine is
:class:`DeviceRankEngine` (libbltc).  The host logic (partition, exchange,
ordering, assembly) is engine-agnostic so it is unit-tested with world-size-2
``gloo`` process groups on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .particles import Points
from .tree_types import BoundingBox

RECORD_DOUBLES = 18   # flattened TreeArray record (csrc/api.cu kRec)


def moment_stride(degree: int) -> int:
    m3 = (degree + 1) ** 3
    return (m3 + 1) & ~1


# ---------------------------------------------------------------------------
# Recursive coordinate bisection (decomp.py:49-130)


@dataclass(eq=False)
class CutNode:
    axis: int
    value: float
    left: "CutNode | int"
    right: "CutNode | int"


@dataclass(eq=False)
class RcbPartition:
    assignment: np.ndarray       # original index -> rank id
    order: np.ndarray            # original indices grouped rank-contiguously
    rank_start: np.ndarray       # length R+1 offsets into order
    regions: list                # rank slabs tiling the root box
    cuts: "CutNode | int"

    def rank_indices(self, rank: int) -> np.ndarray:
        return self.order[self.rank_start[rank]:self.rank_start[rank + 1]]

    @property
    def counts(self) -> np.ndarray:
        return np.diff(self.rank_start)


def _cut_axis(lo: np.ndarray, hi: np.ndarray) -> int:
    return int(np.argmax(hi - lo))   # ties resolve to the lowest axis (decomp.py:71-73)


def rcb_partition(points: Points, ranks: int) -> RcbPartition:
    """Cut the longest extent of the current slab at an exact order statistic;
    ranks split floor/ceil; per-rank counts differ by at most one."""
    n = len(points)
    if ranks < 1:
        raise ValueError("ranks must be >= 1")
    if n < ranks:
        raise ValueError(f"need at least one particle per rank ({n} < {ranks})")
    coords = (np.asarray(points.x), np.asarray(points.y), np.asarray(points.z))
    root_lo = np.array([c.min() for c in coords])
    root_hi = np.array([c.max() for c in coords])
    order = np.arange(n)
    assignment = np.empty(n, dtype=np.int64)
    shares = np.array([(n * (r + 1)) // ranks - (n * r) // ranks for r in range(ranks)],
                      dtype=np.int64)
    regions: list = [None] * ranks

    def recurse(start, stop, r0, r1, lo, hi):
        if r1 - r0 == 1:
            assignment[order[start:stop]] = r0
            regions[r0] = BoundingBox(lo.copy(), hi.copy())
            return r0
        rm = r0 + (r1 - r0) // 2
        n_left = int(shares[r0:rm].sum())
        axis = _cut_axis(lo, hi)
        idx = order[start:stop]
        vals = coords[axis][idx]
        if n_left > 0:
            idx = idx[np.argpartition(vals, n_left - 1)]
            order[start:stop] = idx
        left_max = float(coords[axis][idx[:n_left]].max())
        right_min = float(coords[axis][idx[n_left:]].min())
        cut = 0.5 * (left_max + right_min)
        lo_hi = hi.copy()
        lo_hi[axis] = cut
        hi_lo = lo.copy()
        hi_lo[axis] = cut
        left = recurse(start, start + n_left, r0, rm, lo, lo_hi)
        right = recurse(start + n_left, stop, rm, r1, hi_lo, hi)
        return CutNode(axis=axis, value=cut, left=left, right=right)

    cuts = recurse(0, n, 0, ranks, root_lo, root_hi)
    rank_start = np.concatenate(([0], np.cumsum(shares)))
    return RcbPartition(assignment=assignment, order=order, rank_start=rank_start,
                        regions=regions, cuts=cuts)


class DeviceRcb:
    """RCB on the device (FAST runs): the same cuts, axes and per-rank counts
    as rcb_partition (decomp.py:76-130) -- exact order statistics, floor/ceil
    shares, the longest slab extent, ties to the lowest axis.  Each cut is a
    selection, not a sort: ``torch.kthvalue`` finds the n_left-th and
    (n_left+1)-th smallest coordinates (left_max, right_min), and an
    order-preserving compaction splits the slab at them -- O(n) per cut and
    one small host read (the two order statistics, which also give the cut
    plane).  Each rank gets exactly the reference's particle SET; the order
    within a rank is the input order (the reference's argpartition order
    differs), which only changes FAST summation order.  ``order`` stays on
    the device.  When particles share the coordinate at a cut's order
    statistic the reference's introselect decides which tied particles go
    left: ``tied`` is then True and callers fall back to the host
    rcb_partition."""

    def __init__(self, x, y, z, ranks: int):
        import torch
        n = int(x.numel())
        if ranks < 1:
            raise ValueError("ranks must be >= 1")
        if n < ranks:
            raise ValueError(f"need at least one particle per rank ({n} < {ranks})")
        coords = (x, y, z)
        ext = torch.stack([torch.stack([c.min(), c.max()]) for c in coords]).cpu().numpy()
        lo, hi = ext[:, 0].copy(), ext[:, 1].copy()
        self.order = torch.arange(n, device=x.device)
        self.tied = False
        shares = np.array([(n * (r + 1)) // ranks - (n * r) // ranks for r in range(ranks)],
                          dtype=np.int64)
        self.rank_start = np.concatenate(([0], np.cumsum(shares)))

        def recurse(start, stop, r0, r1, lo, hi):
            if r1 - r0 == 1 or self.tied:
                return
            rm = r0 + (r1 - r0) // 2
            n_left = int(shares[r0:rm].sum())
            axis = _cut_axis(lo, hi)
            idx = self.order[start:stop]
            vals = coords[axis][idx]
            stats = torch.stack([torch.kthvalue(vals, n_left).values,
                                 torch.kthvalue(vals, n_left + 1).values])
            left_max, right_min = (float(v) for v in stats.cpu().tolist())
            if left_max == right_min:
                self.tied = True
                return
            go_left = vals <= left_max   # exactly n_left: no value sits in between
            self.order[start:stop] = torch.cat([idx[go_left], idx[~go_left]])
            cut = 0.5 * (left_max + right_min)
            lo_hi = hi.copy()
            lo_hi[axis] = cut
            hi_lo = lo.copy()
            hi_lo[axis] = cut
            recurse(start, start + n_left, r0, rm, lo, lo_hi)
            recurse(start + n_left, stop, rm, r1, hi_lo, hi)

        recurse(0, n, 0, ranks, lo, hi)

    def rank_indices(self, rank: int):
        return self.order[int(self.rank_start[rank]):int(self.rank_start[rank + 1])]

    @property
    def counts(self) -> np.ndarray:
        return np.diff(self.rank_start)


# ---------------------------------------------------------------------------
# Published rank data and its exchange


@dataclass(eq=False)
class Published:
    """One rank's frozen data (RankWindows, decomp.py:197-208) as flat tensors:
    records [n_clusters, 18], particles [4, n] (x, y, z, q reordered),
    moments [n_rows, moment_stride]."""

    records: object
    particles: object
    moments: object
    block: object = None   # the packed [records | particles | moments] buffer, if any

    @property
    def sizes(self) -> tuple[int, int, int]:
        return (int(self.records.shape[0]), int(self.particles.shape[1]),
                int(self.moments.shape[0]))


# ---------------------------------------------------------------------------
# Collectives.  NCCL moves CUDA tensors directly over NVLink; a gloo group
# (CPU tests, or several ranks sharing one GPU) gets host copies.


def _via_host(t, group) -> bool:
    import torch.distributed as dist
    return t.is_cuda and dist.get_backend(group) == "gloo"


def _all_gather(out_list, t, group=None):
    import torch
    import torch.distributed as dist
    if _via_host(t, group):
        outs = [torch.empty(o.shape, dtype=o.dtype) for o in out_list]
        dist.all_gather(outs, t.cpu(), group=group)
        for o, h in zip(out_list, outs):
            o.copy_(h)
    else:
        dist.all_gather(out_list, t, group=group)


def _all_to_all_single(out, inp, out_split=None, in_split=None, group=None):
    import torch
    import torch.distributed as dist
    if _via_host(inp, group):
        h = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(h, inp.cpu(), out_split, in_split, group=group)
        out.copy_(h)
    else:
        dist.all_to_all_single(out, inp, out_split, in_split, group=group)


def _all_reduce(t, group=None):
    import torch.distributed as dist
    if _via_host(t, group):
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)


def packed_doubles(sizes, ncols: int) -> int:
    """Doubles of one rank's packed publication [records | particles |
    moment rows], rounded up to 32 (256-byte blocks, so every rank's block
    and its moment rows stay aligned inside the gathered buffer)."""
    nc, n, nrow = sizes
    return (nc * RECORD_DOUBLES + 4 * n + nrow * ncols + 31) // 32 * 32


def unpack_published(block, sizes, ncols: int) -> Published:
    """Views of one rank's packed block (layout of ``packed_doubles``)."""
    nc, n, nrow = sizes
    o1 = nc * RECORD_DOUBLES
    o2 = o1 + 4 * n
    return Published(block[:o1].view(nc, RECORD_DOUBLES), block[o1:o2].view(4, n),
                     block[o2:o2 + nrow * ncols].view(nrow, ncols))


def _all_gather_flat(out, buf, ranks: int, group=None):
    """out[ranks * buf.numel()] <- every rank's buf: NCCL's all_gather_into_
    tensor (one collective, no per-rank output list) for CUDA tensors on an
    NCCL group; the list form (host copies for gloo) otherwise."""
    import torch.distributed as dist
    if buf.is_cuda and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        _all_gather(list(out.view(ranks, -1).unbind(0)), buf, group=group)


def domain_boxes(x, y, z, grid: int = 16) -> np.ndarray:
    """The global target set as the minimal bounding boxes of the occupied
    cells of a ``grid``^3 grid over its bounding box ([k, 6]: lo xyz, hi
    xyz; bltc_domain_cells, host only).  Every batch centre lies in one of
    them, so a rank skips the moment rows of clusters no batch in any box
    could accept (bltc_rank_set_domain_boxes) -- on a Plummer sphere the
    top clusters of each rank, whose reach r_C / theta falls into the empty
    corners of the bounding box."""
    import ctypes

    from . import _lib
    f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    x, y, z = f64(x), f64(y), f64(z)
    out = np.empty((grid ** 3, 6), dtype=np.float64)
    nb = ctypes.c_int64(0)
    _lib.check(_lib.load().bltc_domain_cells(len(x), _lib.f64p(x), _lib.f64p(y), _lib.f64p(z),
                                             grid, _lib.f64p(out), ctypes.byref(nb)))
    return out[:nb.value].copy()


def all_gather_sizes(sizes, ranks: int, group=None, device=None) -> list[tuple]:
    """Every rank's (n_clusters, n_particles, n_moment_rows): one tiny
    all-gather, the step's only host read-back of the exchange."""
    import torch
    t = torch.tensor(sizes, dtype=torch.int64, device=device)
    out = torch.empty(ranks * 3, dtype=torch.int64, device=device)
    _all_gather_flat(out, t, ranks, group)
    h = out.view(ranks, 3).tolist()
    return [tuple(int(v) for v in s) for s in h]


def all_gather_published(pub: Published, ranks: int, group=None,
                         all_sizes: list | None = None) -> list[Published]:
    """Replicate every rank's published data on every rank -- north_star's
    single all-gather of the source tree, proxy charges and near-field
    particles: one packed [records | particles | moments] block per rank,
    padded to the largest rank's block, moved by ONE all-gather (NCCL over
    NVLink for CUDA tensors, gloo for CPU tensors).  ``pub`` may already be a
    view of a packed block (DeviceRankEngine.publish_packed); the sizes
    all-gather is skipped when ``all_sizes`` is given."""
    import torch

    dev = pub.records.device
    ncols = int(pub.moments.shape[1])
    if all_sizes is None:
        all_sizes = all_gather_sizes(pub.sizes, ranks, group, dev)
    cap = max(packed_doubles(s, ncols) for s in all_sizes)
    mine = getattr(pub, "block", None)
    if mine is None or mine.numel() != cap:
        buf = torch.zeros(cap, dtype=torch.float64, device=dev)
        nc, n, nrow = pub.sizes
        o1, o2 = nc * RECORD_DOUBLES, nc * RECORD_DOUBLES + 4 * n
        buf[:o1] = pub.records.reshape(-1)
        buf[o1:o2] = pub.particles.reshape(-1)
        buf[o2:o2 + nrow * ncols] = pub.moments.reshape(-1)
        mine = buf
    out = torch.empty(ranks * cap, dtype=torch.float64, device=dev)
    _all_gather_flat(out, mine, ranks, group)
    blocks = out.view(ranks, cap)
    return [unpack_published(blocks[r], all_sizes[r], ncols) for r in range(ranks)]


def all_gather_records(pub: Published, ranks: int, group=None) -> list:
    """LET step one's collective: every rank's tree records on every rank
    (one size all-gather, one padded all-gather)."""
    import torch

    dev = pub.records.device
    n = torch.tensor([pub.records.shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.empty_like(n) for _ in range(ranks)]
    _all_gather(sizes, n, group=group)
    sizes = [int(v.item()) for v in sizes]
    cap = max(1, max(sizes)) * RECORD_DOUBLES
    buf = torch.zeros(cap, dtype=torch.float64, device=dev)
    buf[:pub.records.numel()] = pub.records.reshape(-1)
    gathered = [torch.empty_like(buf) for _ in range(ranks)]
    _all_gather(gathered, buf, group=group)
    return [gathered[r][:sizes[r] * RECORD_DOUBLES].view(sizes[r], RECORD_DOUBLES)
            for r in range(ranks)]


@dataclass(eq=False)
class LetPlan:
    """What one origin fetches from every owner (build_let, decomp.py:366-399):
    per owner the sorted moment-row ids ``a[o]`` and particle-slice ids
    ``d[o]`` (device tensors) and, on the host, their counts, the number of
    clusters in both lists and the particle count of the slices."""

    a: dict
    d: dict
    na: dict
    nd: dict
    nboth: dict
    npart: dict


def let_plan(flags: list, records: list, me: int) -> LetPlan:
    """All owners at once with three host synchronisations (not one per
    owner and list): need flags -> ids, counts and particle totals."""
    import torch
    R = len(flags)
    dev = flags[0].device
    sizes = [int(f.numel()) for f in flags]
    flat = torch.cat([f.to(torch.int64) for f in flags])
    owner = torch.repeat_interleave(torch.arange(R, device=dev),
                                    torch.tensor(sizes, device=dev))
    offs = torch.tensor([0] + sizes[:-1], device=dev).cumsum(0)
    local = torch.arange(flat.numel(), device=dev) - offs[owner]
    remote = owner != me
    a_pos = torch.nonzero(((flat & 1) != 0) & remote).reshape(-1)
    d_pos = torch.nonzero(((flat & 2) != 0) & remote).reshape(-1)
    # particle counts of the direct clusters, from the owners' records
    cnt = torch.cat([r[:, 15] - r[:, 14] for r in records]).to(torch.int64)
    both = ((flat & 3) == 3) & remote
    stats = torch.stack([torch.bincount(owner[a_pos], minlength=R),
                         torch.bincount(owner[d_pos], minlength=R),
                         torch.bincount(owner[both], minlength=R),
                         torch.bincount(owner[d_pos], weights=cnt[d_pos].to(torch.float64),
                                        minlength=R).to(torch.int64)]).cpu()
    na, nd, nb, npart = (stats[i].tolist() for i in range(4))
    a_ids = torch.split(local[a_pos], na)
    d_ids = torch.split(local[d_pos], nd)
    return LetPlan(a={o: a_ids[o] for o in range(R)}, d={o: d_ids[o] for o in range(R)},
                   na=dict(enumerate(na)), nd=dict(enumerate(nd)), nboth=dict(enumerate(nb)),
                   npart=dict(enumerate(npart)))


def let_request(flags) -> tuple:
    """Cluster ids one origin needs from one owner, each sorted ascending as
    in build_let (decomp.py:372-373): (moment-row ids, particle-slice ids)."""
    import torch
    f = flags.to(torch.int64)
    a = torch.nonzero(f & 1).reshape(-1)
    d = torch.nonzero(f & 2).reshape(-1)
    return a, d


def _slice_index(records, d_ids, total: int | None = None):
    """Concatenated particle indices of the clusters d_ids (list order) and
    the slice sizes; ``total`` (the sum of the sizes) avoids a host sync."""
    import torch
    dev = records.device
    if d_ids.numel() == 0:
        z = torch.zeros(0, dtype=torch.int64, device=dev)
        return z, z
    st = records[d_ids, 14].to(torch.int64)
    sz = records[d_ids, 15].to(torch.int64) - st
    off = torch.cumsum(sz, 0) - sz
    if total is None:
        total = int(sz.sum().item())
    seg = torch.repeat_interleave(torch.arange(d_ids.numel(), device=dev), sz,
                                  output_size=total)
    idx = st[seg] + (torch.arange(total, device=dev) - off[seg])
    return idx, sz


def let_serve(pub: Published, a_ids, d_ids, npart: int | None = None):
    """Owner side of step two: the requested moment rows and particle slices,
    flattened into one float64 buffer (rows first)."""
    import torch
    mrow = pub.records[a_ids, 16].to(torch.int64)
    rows = pub.moments[mrow] if a_ids.numel() else pub.moments[:0]
    idx, _ = _slice_index(pub.records, d_ids, npart)
    par = pub.particles[:, idx]
    return torch.cat([rows.reshape(-1), par.reshape(-1)])


def let_serve_many(pub: Published, requests: list):
    """let_serve for several requesters [(a_ids, d_ids) | None] with one host
    synchronisation for all their particle totals."""
    import torch
    live = [i for i, r in enumerate(requests) if r is not None and r[1].numel()]
    totals = {}
    if live:
        sums = torch.stack([(pub.records[requests[i][1], 15]
                             - pub.records[requests[i][1], 14]).sum() for i in live]).cpu()
        totals = {i: int(v) for i, v in zip(live, sums.tolist())}
    return [None if r is None else let_serve(pub, r[0], r[1], totals.get(i, 0))
            for i, r in enumerate(requests)]


def let_payload_size(records, a_ids, d_ids, ncols: int) -> int:
    import torch
    p = 0
    if d_ids.numel():
        p = int((records[d_ids, 15] - records[d_ids, 14]).to(torch.int64).sum().item())
    return int(a_ids.numel()) * ncols + 4 * p


def let_assemble(records, a_ids, d_ids, payload, ncols: int, npart: int | None = None,
                 nboth: int | None = None):
    """Origin side of step two: the owner's fetched data as a Published whose
    records point into the fetched buffers (moment row -> index among the
    fetched rows, particle range -> offset in the fetched slices; records of
    clusters not fetched keep no data).  Returns (Published, FetchStats)."""
    import torch
    na = int(a_ids.numel())
    rows = payload[:na * ncols].view(na, ncols)
    sz = (records[d_ids, 15] - records[d_ids, 14]).to(torch.int64)
    P = int(sz.sum().item()) if npart is None else int(npart)
    par = payload[na * ncols:na * ncols + 4 * P].view(4, P)
    rec = records.clone()
    rec[:, 14] = 0.0
    rec[:, 15] = 0.0
    rec[:, 16] = -1.0
    if na:
        rec[a_ids, 16] = torch.arange(na, dtype=rec.dtype, device=rec.device)
    if d_ids.numel():
        off = torch.cumsum(sz, 0) - sz
        rec[d_ids, 14] = off.to(rec.dtype)
        rec[d_ids, 15] = (off + sz).to(rec.dtype)
    if nboth is None:
        nboth = int(a_ids.numel() + d_ids.numel()
                    - torch.unique(torch.cat([a_ids, d_ids])).numel())
    fs = FetchStats(tree_records=int(records.shape[0]),
                    clusters=na + int(d_ids.numel()) - int(nboth), moments=na, particles=P)
    return Published(rec, par, rows), fs


def let_exchange(pub: Published, needs_fn, ranks: int, me: int, group=None):
    """Both LET steps over a process group (NCCL for CUDA tensors): returns
    (forest in owner order -- own data for ``me``, fetched data otherwise --
    and {(me, owner): FetchStats})."""
    import torch

    dev = pub.records.device
    ncols = int(pub.moments.shape[1])
    records = all_gather_records(pub, ranks, group)
    plan = let_plan(needs_fn(records), records, me)
    # requests: counts, then ids
    cnt = torch.tensor([[plan.na[o], plan.nd[o]] if o != me else [0, 0] for o in range(ranks)],
                       dtype=torch.int64, device=dev)
    rcnt = torch.empty_like(cnt)
    _all_to_all_single(rcnt, cnt, group=group)
    rcnt_h = rcnt.cpu().tolist()
    send_ids = torch.cat([torch.cat([plan.a[o], plan.d[o]]) for o in range(ranks)])
    in_split = [plan.na[o] + plan.nd[o] if o != me else 0 for o in range(ranks)]
    out_split = [sum(c) for c in rcnt_h]
    recv_ids = torch.empty(sum(out_split), dtype=torch.int64, device=dev)
    _all_to_all_single(recv_ids, send_ids, out_split, in_split, group=group)
    # serve every requester
    reqs, pos = [], 0
    for r in range(ranks):
        na, nd = rcnt_h[r]
        ids = recv_ids[pos:pos + na + nd]
        pos += na + nd
        reqs.append(None if (r == me or na + nd == 0) else (ids[:na], ids[na:]))
    bufs = let_serve_many(pub, reqs)
    serve_split = [0 if b is None else int(b.numel()) for b in bufs]
    live = [b for b in bufs if b is not None]
    send = torch.cat(live) if live else torch.zeros(0, dtype=torch.float64, device=dev)
    fetch_split = [plan.na[o] * ncols + 4 * plan.npart[o] if o != me else 0
                   for o in range(ranks)]
    recv = torch.empty(sum(fetch_split), dtype=torch.float64, device=dev)
    _all_to_all_single(recv, send, fetch_split, serve_split, group=group)
    forest, fetch, pos = [], {}, 0
    for o in range(ranks):
        if o == me:
            forest.append(pub)
            continue
        payload = recv[pos:pos + fetch_split[o]]
        pos += fetch_split[o]
        p_o, fs = let_assemble(records[o], plan.a[o], plan.d[o], payload, ncols,
                               plan.npart[o], plan.nboth[o])
        forest.append(p_o)
        fetch[(me, o)] = fs
    return forest, fetch


def let_local(pubs: dict, needs_fns: dict, ranks: int):
    """Both LET steps for ranks simulated in one process (no process group):
    the same plan / serve / assemble path, handed over in place."""
    ncols = int(pubs[0].moments.shape[1])
    records = [pubs[r].records for r in range(ranks)]
    forests, fetch = {}, {}
    for me in range(ranks):
        plan = let_plan(needs_fns[me](records), records, me)
        forest = []
        for o in range(ranks):
            if o == me:
                forest.append(pubs[me])
                continue
            payload = let_serve(pubs[o], plan.a[o], plan.d[o], plan.npart[o])
            p_o, fs = let_assemble(records[o], plan.a[o], plan.d[o], payload, ncols,
                                   plan.npart[o], plan.nboth[o])
            forest.append(p_o)
            fetch[(me, o)] = fs
        forests[me] = forest
    return forests, fetch


def let_violations(forest: list, flags: list, me: int) -> dict:
    """decomp.py:402-418: sufficiency (a referenced cluster without its data)
    and minimality (data fetched that no batch references), from one origin's
    fetched forest and its need flags."""
    import torch
    suff = mini = 0
    for o, p in enumerate(forest):
        if o == me:
            continue
        f = flags[o].to(torch.int64)
        has_row = p.records[:, 16] >= 0
        has_par = p.records[:, 15] > p.records[:, 14]
        need_a = (f & 1) != 0
        need_d = ((f & 2) != 0) & (p.records[:, 10] > 0)
        suff += int((need_a & ~has_row).sum().item()) + int((need_d & ~has_par).sum().item())
        mini += int((has_row & ~need_a).sum().item()) + int((has_par & ~need_d).sum().item())
    return {"sufficiency": suff, "minimality": mini}


# ---------------------------------------------------------------------------
# The product rank engine: libbltc on one CUDA device


_rank_ctx: dict = {}


def rank_context(slot: int):
    """A libbltc context for rank slot ``slot`` on the current device and
    torch stream, kept across run_distributed calls: creating and destroying
    a context costs ~0.2 s (device allocations / frees), more than a 1M-
    particle rank's evaluation.  ``release_rank_contexts()`` frees them."""
    import torch

    from .engine import Context
    dev = torch.cuda.current_device()
    stream = torch.cuda.current_stream(dev).cuda_stream
    key = (dev, stream, int(slot))
    ctx = _rank_ctx.get(key)
    if ctx is None:
        ctx = _rank_ctx[key] = Context(dev, stream)
    return ctx


def release_rank_contexts() -> None:
    for ctx in _rank_ctx.values():
        ctx.close()
    _rank_ctx.clear()


class DeviceRankEngine:
    """One rank's device pipeline (bltc_rank_build / _publish / _evaluate)."""

    def __init__(self, config, mode: str | None = None, device: int | None = None,
                 context=None):
        import torch

        from .engine import Context, make_params
        self.torch = torch
        self.device = torch.cuda.current_device() if device is None else int(device)
        # libbltc runs on torch's current stream, so the tensors this engine
        # hands it (inputs, exchanged buffers) are stream-ordered with it
        self.ctx = context or Context(self.device,
                                      torch.cuda.current_stream(self.device).cuda_stream)
        self.params = make_params(config, mode, all_moments=False)
        self.n = 0
        self.stats = None

    def set_domain(self, lo, hi) -> None:
        """The bounding box of ALL ranks' targets: moment rows no batch in it
        could read are not computed or published (bltc_rank_set_domain)."""
        self.set_domain_boxes(np.concatenate([np.asarray(lo, dtype=np.float64),
                                              np.asarray(hi, dtype=np.float64)]))

    def set_domain_boxes(self, boxes) -> None:
        """ALL ranks' targets as a union of boxes ([k, 6], e.g. domain_boxes):
        the tighter form of set_domain (bltc_rank_set_domain_boxes)."""
        self.domain = np.ascontiguousarray(boxes, dtype=np.float64).reshape(-1, 6)

    def build(self, x, y, z, q) -> None:
        torch = self.torch
        dev = torch.device("cuda", self.device)
        dom = getattr(self, "domain", None)
        self.ctx.rank_set_domain_boxes(dom if dom is not None else np.empty((0, 6)))
        self._inputs = [torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64)
                                        if not isinstance(v, torch.Tensor) else v,
                                        device=dev).contiguous() for v in (x, y, z, q)]
        self.n = int(self._inputs[0].shape[0])
        self._sync()
        self.ctx.rank_build(self.params, self.n, *[t.data_ptr() for t in self._inputs],
                            device_ptrs=True)

    def publish(self) -> Published:
        torch = self.torch
        sz = self.ctx.rank_publish_sizes()
        dev = torch.device("cuda", self.device)
        rec = torch.empty((sz["n_clusters"], RECORD_DOUBLES), dtype=torch.float64, device=dev)
        par = torch.empty((4, sz["n_particles"]), dtype=torch.float64, device=dev)
        mom = torch.empty((max(1, sz["n_moment_rows"]), moment_stride(self.params.degree)),
                          dtype=torch.float64, device=dev)
        self._sync()
        self.ctx.rank_publish(rec.data_ptr(), par.data_ptr(), mom.data_ptr())
        self._sync_after()
        return Published(rec, par, mom[:sz["n_moment_rows"]])

    def publish_sizes(self) -> tuple:
        sz = self.ctx.rank_publish_sizes()
        return (int(sz["n_clusters"]), int(sz["n_particles"]), int(sz["n_moment_rows"]))

    def publish_packed(self, cap: int) -> Published:
        """Publish straight into one packed block of ``cap`` doubles
        (decomp.packed_doubles layout), ready for all_gather_published's
        single collective: no staging copies."""
        torch = self.torch
        sizes = self.publish_sizes()
        ncols = moment_stride(self.params.degree)
        block = torch.empty(cap, dtype=torch.float64, device=torch.device("cuda", self.device))
        pub = unpack_published(block, sizes, ncols)
        pub.block = block
        self._sync()
        # zero-row moment views still need a valid pointer (nothing is written)
        mom_ptr = pub.moments.data_ptr() if sizes[2] else block.data_ptr()
        self.ctx.rank_publish(pub.records.data_ptr(), pub.particles.data_ptr(), mom_ptr)
        self._sync_after()
        return pub

    def _same_stream(self) -> bool:
        cur = self.torch.cuda.current_stream(self.device).cuda_stream
        return getattr(self.ctx, "stream", None) == cur

    def _sync(self):
        """Order torch's work before libbltc's when the context has its own
        stream (a caller-supplied context); nothing to do when libbltc runs
        on torch's current stream (the rank contexts, the bench)."""
        if not self._same_stream():
            self.torch.cuda.current_stream(self.device).synchronize()

    def _sync_after(self):
        """Order libbltc's work before torch's (collectives on the published
        buffers) when the context has its own stream."""
        if not self._same_stream():
            self.torch.cuda.synchronize(self.device)

    def needs(self, ranks: int, my_rank: int, records: list) -> list:
        """LET step one on the device: per owner, int32 need flags per cluster."""
        torch = self.torch
        dev = torch.device("cuda", self.device)
        sizes = [int(r.shape[0]) for r in records]
        recs = [r.to(dev).contiguous() for r in records]
        flags = torch.empty(max(1, sum(sizes)), dtype=torch.int32, device=dev)
        self._sync()
        self.ctx.rank_needs(self.params, ranks, my_rank, sizes, [r.data_ptr() for r in recs],
                            flags.data_ptr())
        out, pos = [], 0
        for n in sizes:
            out.append(flags[pos:pos + n])
            pos += n
        return out

    def evaluate(self, ranks: int, my_rank: int, forest: list[Published]):
        torch = self.torch
        dev = torch.device("cuda", self.device)
        phi = torch.empty(self.n, dtype=torch.float64, device=dev)
        sizes = [p.sizes for p in forest]
        # zero-row moment tensors still need a valid pointer
        mom_ptrs = [p.moments.data_ptr() if p.moments.numel() else p.records.data_ptr()
                    for p in forest]
        self._sync()
        self.stats = self.ctx.rank_evaluate(
            self.params, ranks, my_rank, [s[0] for s in sizes], [s[1] for s in sizes],
            [s[2] for s in sizes], [p.records.data_ptr() for p in forest],
            [p.particles.data_ptr() for p in forest], mom_ptrs, phi.data_ptr(),
            device_ptrs=True)
        return phi


# ---------------------------------------------------------------------------
# Orchestration


@dataclass(eq=False)
class FetchStats:
    """Per (origin, owner) exchange volume (decomp.py:324-331): the reference's
    LET counts with exchange="let"; with "replicate" every origin receives
    the owner's whole tree."""

    tree_records: int = 0
    clusters: int = 0
    moments: int = 0
    particles: int = 0


@dataclass(eq=False)
class RankTimings:
    rank: int
    tree_s: float
    moments_s: float
    let_s: float
    eval_s: float


@dataclass(eq=False)
class DistributedStats:
    n_ranks: int
    rank_counts: np.ndarray
    n_clusters: int
    n_batches: int
    direct_pairs: int
    approx_pairs: int
    fetch_stats: dict = field(default_factory=dict)
    rank_timings: list = field(default_factory=list)
    setup_s: float = 0.0
    precompute_s: float = 0.0
    compute_s: float = 0.0
    total_s: float = 0.0


def _process_group_world(group):
    try:
        import torch.distributed as dist
    except ImportError:
        return None, 1, 0
    if not (dist.is_available() and dist.is_initialized()):
        return None, 1, 0
    return dist, dist.get_world_size(group), dist.get_rank(group)


def run_distributed(system, config, ranks: int, threads: int = 1, mode: str | None = None,
                    group=None, engine_factory=None, exchange: str = "let",
                    partition: str = "auto"):
    """decomp.py:483-593 on GPUs.  Returns (phi in original order, stats) on
    every participating process.  ``threads`` is accepted and ignored;
    ``exchange`` is "let" (the reference's minimal fetch) or "replicate";
    ``partition`` "host" is the reference's numpy RCB (its exact particle
    order, needed for bitwise PARITY), "device" the same cuts on the GPU
    (DeviceRcb), "auto" = device for FAST runs on the device engine."""
    import time

    import torch

    from .engine import DEFAULT_MODE

    del threads
    if exchange not in ("let", "replicate"):
        raise ValueError(f"exchange must be 'let' or 'replicate', got {exchange!r}")
    if partition not in ("auto", "host", "device"):
        raise ValueError(f"partition must be 'auto', 'host' or 'device', got {partition!r}")
    if not system.coincident:
        raise ValueError("distributed runs require targets and sources "
                         "to be the same particle set")
    t_start = time.perf_counter()
    resolved = DEFAULT_MODE if mode is None else mode
    on_device = partition == "device" or (partition == "auto" and engine_factory is None
                                          and resolved == "fast")
    dist, world, me = _process_group_world(group)
    if world > 1 and world != ranks:
        raise ValueError(f"ranks ({ranks}) must equal the process-group size ({world})")
    mine = [me] if world > 1 else list(range(ranks))
    if engine_factory is not None:
        engines = {r: engine_factory() for r in mine}
    else:
        engines = {r: DeviceRankEngine(config, mode, context=rank_context(r)) for r in mine}
    src = system.sources
    x, y, z = np.asarray(src.x), np.asarray(src.y), np.asarray(src.z)
    q = np.asarray(system.charges)
    if len(x):
        boxes = domain_boxes(x, y, z)
        for e in engines.values():
            if hasattr(e, "set_domain_boxes"):
                e.set_domain_boxes(boxes)
            elif hasattr(e, "set_domain"):
                e.set_domain(boxes[:, :3].min(axis=0), boxes[:, 3:].max(axis=0))
    if on_device:
        dev = torch.device("cuda", torch.cuda.current_device())
        x, y, z, q = (torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(dev)
                      for v in (x, y, z, q))
        part = DeviceRcb(x, y, z, ranks)
        if part.tied:   # ties at a cut: the reference's own partition
            x, y, z, q = (np.asarray(v) for v in (src.x, src.y, src.z, system.charges))
            part = rcb_partition(system.sources, ranks)
    else:
        part = rcb_partition(system.sources, ranks)
    timings = {}
    t0 = time.perf_counter()
    for r in mine:
        idx = part.rank_indices(r)
        tr = time.perf_counter()
        engines[r].build(x[idx], y[idx], z[idx], q[idx])
        timings[r] = [time.perf_counter() - tr, 0.0, 0.0, 0.0]
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    pubs = {r: engines[r].publish() for r in mine}
    fetch = {}
    if exchange == "let" and world > 1:
        f, fetch = let_exchange(pubs[me], lambda recs: engines[me].needs(ranks, me, recs),
                                ranks, me, group)
        forests = {me: f}
    elif exchange == "let":
        needs = {r: (lambda recs, r=r: engines[r].needs(ranks, r, recs)) for r in mine}
        forests, fetch = let_local(pubs, needs, ranks)
    elif world > 1:
        forests = {me: all_gather_published(pubs[me], ranks, group)}
    else:
        forests = {r: [pubs[o] for o in range(ranks)] for r in mine}
    t_exchange = time.perf_counter() - t0
    for r in mine:
        timings[r][2] = t_exchange
    t0 = time.perf_counter()
    rank_phi = {}
    for r in mine:
        tr = time.perf_counter()
        rank_phi[r] = engines[r].evaluate(ranks, r, forests[r])
        timings[r][3] = time.perf_counter() - tr
    t_eval = time.perf_counter() - t0

    phi = np.empty(len(system.targets))
    local = np.zeros(4, dtype=np.int64)   # direct, approx, clusters, batches
    for r in mine:
        st = engines[r].stats
        local += [st.direct_pairs, st.approx_pairs, st.n_clusters, st.n_batches]
    if world > 1:
        dev = pubs[me].records.device
        counts = part.counts
        cap = int(counts.max())
        buf = torch.zeros(cap, dtype=torch.float64, device=dev)
        mine_phi = rank_phi[me].reshape(-1)
        buf[:mine_phi.numel()] = mine_phi
        gathered = [torch.empty_like(buf) for _ in range(ranks)]
        _all_gather(gathered, buf, group=group)
        rank_phi = {o: gathered[o][:counts[o]] for o in range(ranks)}
        tot = torch.tensor(local, dtype=torch.int64, device=dev)
        _all_reduce(tot, group=group)
        local = tot.cpu().numpy()
    if on_device:
        full = torch.empty(len(system.targets), dtype=torch.float64, device=x.device)
        for o in range(ranks):
            full[part.rank_indices(o)] = rank_phi[o].reshape(-1).to(x.device)
        phi = full.cpu().numpy()
    else:
        for o in range(ranks):
            phi[part.rank_indices(o)] = rank_phi[o].detach().reshape(-1).cpu().numpy()
    if exchange == "replicate":
        for r in mine:
            for o in range(ranks):
                if o != r:
                    nc, n, nrow = forests[r][o].sizes
                    fetch[(r, o)] = FetchStats(tree_records=nc, clusters=nc, moments=nrow,
                                               particles=n)
    total = time.perf_counter() - t_start
    stats = DistributedStats(
        n_ranks=ranks, rank_counts=part.counts, n_clusters=int(local[2]),
        n_batches=int(local[3]), direct_pairs=int(local[0]), approx_pairs=int(local[1]),
        fetch_stats=fetch,
        rank_timings=[RankTimings(r, *timings[r]) for r in mine],
        setup_s=t_build + t_exchange, precompute_s=0.0, compute_s=t_eval, total_s=total)
    return phi, stats


class DeviceRankRunner:
    """One rank of a one-process-per-GPU run with device-resident inputs:
    the RCB partition is computed once (the paper also partitions outside the
    timed region); each ``step()`` is a full distributed
    evaluation -- local tree / batches / moments, the forest all-gather over
    NCCL, evaluation of the local batches -- and returns the rank's stats."""

    def __init__(self, ctx, system, config, mode: str | None = None, group=None,
                 exchange: str = "replicate"):
        import torch
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.ranks = dist.get_world_size(group)
        self.me = dist.get_rank(group)
        part = rcb_partition(system.sources, self.ranks)
        idx = part.rank_indices(self.me)
        src = system.sources
        dev = torch.device("cuda", torch.cuda.current_device())
        self.inputs = [torch.from_numpy(np.ascontiguousarray(np.asarray(a)[idx])).to(dev)
                       for a in (src.x, src.y, src.z, system.charges)]
        self.engine = DeviceRankEngine(config, mode, context=ctx)
        self.engine.set_domain_boxes(domain_boxes(src.x, src.y, src.z))
        self.n_local = int(idx.shape[0])
        self.exchange = exchange
        self.phi = None
        self.fetch = {}

    def step(self):
        self.engine.build(*self.inputs)
        if self.exchange == "let":
            pub = self.engine.publish()
            forest, self.fetch = let_exchange(
                pub, lambda recs: self.engine.needs(self.ranks, self.me, recs), self.ranks,
                self.me, self.group)
        else:
            # north_star's exchange: one sizes all-gather (a few bytes), then
            # ONE all-gather of every rank's packed tree / particles / moments
            all_sizes = all_gather_sizes(self.engine.publish_sizes(), self.ranks, self.group,
                                         self.inputs[0].device)
            ncols = moment_stride(self.engine.params.degree)
            pub = self.engine.publish_packed(max(packed_doubles(s, ncols) for s in all_sizes))
            forest = all_gather_published(pub, self.ranks, self.group, all_sizes=all_sizes)
        self.phi = self.engine.evaluate(self.ranks, self.me, forest)
        return self.engine.stats


def run_distributed_native(system, config, ranks: int, devices=None, mode: str | None = None):
    """run_distributed (decomp.py:483-593) through the single C call
    ``bltc_run_distributed``: R ranks in this process on ``devices`` (rank r
    on devices[r % len(devices)], default: every visible GPU), the
    reference's host RCB (rcb_partition) fixing each rank's particles and
    order.  No torch.distributed; ranks read each other's published trees
    across devices.  Returns (phi in original order, DistributedStats)."""
    import ctypes
    import time

    from . import _lib
    from .engine import cheb_nodes, make_params

    if not system.coincident:
        raise ValueError("distributed runs require targets and sources "
                         "to be the same particle set")
    if ranks < 1:
        raise ValueError("ranks must be >= 1")
    if devices is None:
        import torch
        devices = list(range(max(1, torch.cuda.device_count())))
    devices = np.ascontiguousarray(devices, dtype=np.int32)
    t0 = time.perf_counter()
    src = system.sources
    part = rcb_partition(src, ranks)
    counts = np.diff(part.rank_start)
    if (counts < 1).any():
        raise ValueError("every rank needs at least one particle")
    p = make_params(config, mode)
    s = cheb_nodes(int(config.degree))
    f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    x, y, z, q = f64(src.x), f64(src.y), f64(src.z), f64(system.charges)
    order = np.ascontiguousarray(part.order, dtype=np.int64)
    start = np.ascontiguousarray(part.rank_start, dtype=np.int64)
    n = len(x)
    phi = np.empty(n)
    st = _lib.Stats()
    dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    ip = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    _lib.check(_lib.load().bltc_run_distributed(
        ranks, devices.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(devices),
        ctypes.byref(p), dp(s), n, dp(x), dp(y), dp(z), dp(q), ip(order), ip(start), dp(phi),
        ctypes.byref(st)))
    return phi, DistributedStats(
        n_ranks=ranks, rank_counts=counts, n_clusters=int(st.n_clusters),
        n_batches=int(st.n_batches), direct_pairs=int(st.direct_pairs),
        approx_pairs=int(st.approx_pairs), setup_s=float(st.setup_s),
        compute_s=float(st.compute_s), total_s=time.perf_counter() - t0)

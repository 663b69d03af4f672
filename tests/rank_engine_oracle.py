"""A rank engine backed by the CPU oracle -- TEST INFRASTRUCTURE ONLY.

It implements the same build / publish / evaluate interface (and the same
18-double record layout) as the product's DeviceRankEngine, so the host-side
distributed logic of paper_2003_01836_b200.decomp -- RCB, the all-gather of
published buffers, the owner order of the evaluation, the assembly of the
result -- can be exercised with gloo process groups on CPU.
"""
import numpy as np
import torch

from oracle import oracle as orc
from paper_2003_01836_b200.decomp import RECORD_DOUBLES, Published, moment_stride


class OracleRankEngine:
    def __init__(self, config):
        self.cfg = config
        self.stats = None

    def build(self, x, y, z, q):
        c = self.cfg
        self.tree = orc.build_source_tree(x, y, z, q, c.leaf_size)
        if c.batch_size == c.leaf_size:
            t = self.tree
            lf = t.leaf_dfs
            self.batches = orc.Batches(tree=t, start=t.start[lf], stop=t.stop[lf],
                                       center=t.center[lf], radius=t.radius[lf])
        else:
            self.batches = orc.build_target_batches(x, y, z, c.batch_size)
        m3 = (c.degree + 1) ** 3
        which = np.nonzero(self.tree.eligible & (self.tree.count > m3))[0]
        self.rows, self.mrow = orc.compute_moments(self.tree, c.degree, which)

    def publish(self):
        t = self.tree
        nc = t.n_nodes
        rec = np.zeros((nc, RECORD_DOUBLES))
        rec[:, 0:3] = t.lo
        rec[:, 3:6] = t.hi
        rec[:, 6:9] = t.center
        rec[:, 9] = t.radius
        rec[:, 10] = t.count
        rec[:, 11] = np.where(t.child_count > 0, t.child_start, -1)
        rec[:, 12] = t.child_count
        rec[:, 13] = t.eligible
        rec[:, 14] = t.start
        rec[:, 15] = t.stop
        rec[:, 16] = self.mrow
        par = np.stack([t.x, t.y, t.z, t.q])
        ms = moment_stride(self.cfg.degree)
        mom = np.zeros((self.rows.shape[0], ms))
        mom[:, :self.rows.shape[1]] = self.rows
        return Published(torch.from_numpy(rec), torch.from_numpy(par), torch.from_numpy(mom))

    @staticmethod
    def _tree_from(pub, degree):
        rec = pub.records.numpy()
        par = pub.particles.numpy()
        nc = rec.shape[0]
        cs = rec[:, 11].astype(np.int64)
        t = orc.Tree(order=np.zeros(0, np.int64), perm=np.zeros(0, np.int64),
                     start=rec[:, 14].astype(np.int64), stop=rec[:, 15].astype(np.int64),
                     lo=rec[:, 0:3].copy(), hi=rec[:, 3:6].copy(),
                     child_start=np.where(cs < 0, 0, cs), child_count=rec[:, 12].astype(np.int64),
                     depth=np.zeros(nc, np.int32), leaf_dfs=np.zeros(0, np.int64),
                     center=rec[:, 6:9].copy(), radius=rec[:, 9].copy(),
                     x=par[0].copy(), y=par[1].copy(), z=par[2].copy(), q=par[3].copy())
        m3 = (degree + 1) ** 3
        rows = pub.moments.numpy()[:, :m3].copy()
        mrow = rec[:, 16].astype(np.int64)
        return t, rows, mrow

    def needs(self, ranks, my_rank, records):
        """LET step one: need flags per cluster of every owner's tree."""
        c = self.cfg
        out = []
        for o in range(ranks):
            rec = records[o].numpy()
            t = self._tree_geometry(rec)
            lists = orc.build_lists(self.batches, t, c.theta, c.degree)
            f = np.zeros(rec.shape[0], dtype=np.int32)
            f[np.unique(lists.a_idx)] |= 1
            f[np.unique(lists.d_idx)] |= 2
            out.append(torch.from_numpy(f))
        return out

    @staticmethod
    def _tree_geometry(rec):
        nc = rec.shape[0]
        cs = rec[:, 11].astype(np.int64)
        z = np.zeros(0)
        # the MAC reads the record's count (field 10); particle ranges may have
        # been remapped by the LET exchange
        return orc.Tree(order=np.zeros(0, np.int64), perm=np.zeros(0, np.int64),
                        start=np.zeros(nc, np.int64), stop=rec[:, 10].astype(np.int64),
                        lo=rec[:, 0:3].copy(), hi=rec[:, 3:6].copy(),
                        child_start=np.where(cs < 0, 0, cs),
                        child_count=rec[:, 12].astype(np.int64), depth=np.zeros(nc, np.int32),
                        leaf_dfs=np.zeros(0, np.int64), center=rec[:, 6:9].copy(),
                        radius=rec[:, 9].copy(), x=z, y=z, z=z, q=z)

    def evaluate(self, ranks, my_rank, forest):
        c = self.cfg
        owners = [my_rank] + [o for o in range(ranks) if o != my_rank]
        groups = []
        direct = approx = 0
        for o in owners:
            t, rows, mrow = self._tree_from(forest[o], c.degree)
            tg = self._tree_geometry(forest[o].records.numpy())
            lists = orc.build_lists(self.batches, tg, c.theta, c.degree)
            d, a = orc.count_pairs(lists, self.batches, tg.count, c.degree)
            direct += d
            approx += a
            groups.append(orc.SourceGroup(t, rows, mrow, lists))
        out, carry = orc.evaluate(self.batches, groups, c.degree, c.kernel.code, c.kernel.kappa)

        class _S:
            pass
        self.stats = _S()
        self.stats.direct_pairs, self.stats.approx_pairs = direct, approx
        self.stats.n_clusters, self.stats.n_batches = self.tree.n_nodes, self.batches.nb
        return torch.from_numpy((out + carry)[self.batches.tree.perm])

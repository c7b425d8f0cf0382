"""Test-side stand-in for dist.CudaStages: the same staged decomposition
(degree relabel; per-root triangles, 4-cycles, diamonds, 4-cliques; two
integer exchanges; row-block epilogue) written independently in numpy/Python
for small graphs, so the multi-rank orchestration in
paper_2007_11111_b200/dist.py can be exercised under gloo on CPU. It also
serves as an independent check of the root decomposition itself: its result
must equal the oracle's.
"""
import itertools

import numpy as np
import torch

from oracle import binding as ob


class NumpyStages:
    def prepare(self, rp_t, ci_t, n, nnz, mask, lenient):
        rp = rp_t.cpu().numpy().astype(np.int64)
        ci = ci_t.cpu().numpy().astype(np.int64)
        self.n, self.nnz, self.mask, self.lenient = n, nnz, mask | 3, lenient
        deg = np.diff(rp)
        self.perm = np.lexsort((np.arange(n), deg))  # new -> old
        self.inv = np.empty(n, np.int64)
        self.inv[self.perm] = np.arange(n)
        self.adj = [sorted(int(self.inv[x]) for x in ci[rp[o]:rp[o + 1]]) for o in self.perm]
        self.adjs = [set(a) for a in self.adj]
        self.nrp = np.zeros(n + 1, np.int64)
        self.nrp[1:] = np.cumsum([len(a) for a in self.adj])
        self.pos = {}
        for r, a in enumerate(self.adj):
            for k, v in enumerate(a):
                self.pos[(r, v)] = int(self.nrp[r]) + k
        self.C3 = torch.zeros(max(nnz, 0), dtype=torch.int32)
        self.vec = torch.zeros(3 * n, dtype=torch.int64)

    def bounds(self, world):
        return np.array([self.n * r // world for r in range(world + 1)], dtype=np.int64)

    def _canon(self, a, b):
        return self.pos[(min(a, b), max(a, b))]

    def triangles(self, u0, u1):
        c = np.zeros(self.nnz, np.int64)
        for u in range(u0, u1):
            S = [v for v in self.adj[u] if v > u]
            for a, b in itertools.combinations(S, 2):
                if b in self.adjs[a]:
                    c[self._canon(u, a)] += 1
                    c[self._canon(u, b)] += 1
                    c[self._canon(a, b)] += 1
        self.C3 = torch.from_numpy(c.astype(np.int32))
        return self.C3

    def local(self):
        c = self.C3.numpy().astype(np.int64)
        n = self.n
        self.c3full = {}
        for r in range(n):
            for v in self.adj[r]:
                self.c3full[(r, v)] = int(c[self._canon(r, v)])
        self.C3vals = c

    def local_part(self, part, nparts, phase):
        """Row-partitioned sweeps (rows r = part mod nparts). Phase 0: c3, d14,
        d10, p3 of my rows, returns the c3 vector to sum over ranks; phase 1:
        d9 of my rows from the summed c3."""
        n = self.n
        sat = lambda a, b: a - b if a > b else 0  # noqa: E731
        deg = [len(a) for a in self.adj]
        if phase == 0:
            self.local()
            self.partial = nparts > 1
            self.c3v = torch.zeros(n, dtype=torch.int64)
            self.loc = np.zeros((4, n), np.int64)  # d14, d10, p3, d9
            p2 = [sat(sum(deg[v] for v in self.adj[r]), deg[r]) for r in range(n)]
            for r in range(part, n, nparts):
                cc = [self.c3full[(r, x)] for x in self.adj[r]]
                c3 = sum(cc) // 2
                self.c3v[r] = c3
                self.loc[0, r] = sum(c * (c - 1) // 2 for c in cc)
                self.loc[1, r] = sum(c * sat(deg[x], 2) for c, x in zip(cc, self.adj[r]))
                self.loc[2, r] = sat(sum(p2[x] for x in self.adj[r]),
                                     deg[r] * sat(deg[r], 1) + 2 * c3)
            return self.c3v if nparts > 1 else torch.zeros(0, dtype=torch.int64)
        c3 = self.c3v.numpy()
        for r in range(part, n, nparts):
            self.loc[3, r] = sat(sum(int(c3[x]) for x in self.adj[r]), 2 * int(c3[r]))
        return torch.zeros(0, dtype=torch.int64)

    def roots(self, u0, u1):
        n = self.n
        c4 = np.zeros(n, np.int64)
        d13 = np.zeros(n, np.int64)
        d15 = np.zeros(n, np.int64)
        for u in range(u0, u1):
            # 4-cycles with u the highest vertex
            L = {}
            low = [v for v in self.adj[u] if v < u]
            for v in low:
                for w in self.adj[v]:
                    if w < u:
                        L[w] = L.get(w, 0) + 1
            for w, l in L.items():
                pairs = l * (l - 1) // 2
                c4[u] += pairs
                c4[w] += pairs
            for v in low:
                c4[v] += sum(L[w] - 1 for w in self.adj[v] if w < u)
            # triangles / 4-cliques with u the lowest vertex
            S = [v for v in self.adj[u] if v > u]
            for a, b in itertools.combinations(S, 2):
                if b in self.adjs[a]:
                    d13[u] += self.c3full[(a, b)] - 1
                    d13[a] += self.c3full[(u, b)] - 1
                    d13[b] += self.c3full[(u, a)] - 1
            for a, b, x in itertools.combinations(S, 3):
                if b in self.adjs[a] and x in self.adjs[a] and x in self.adjs[b]:
                    for y in (u, a, b, x):
                        d15[y] += 1
        if getattr(self, "partial", False):  # 7n: d14 d10 p3 d9 | c4 d13 d15
            self.vec = torch.from_numpy(np.concatenate([self.loc.reshape(-1), c4, d13, d15]))
        else:
            self.vec = torch.from_numpy(np.concatenate([c4, d13, d15]))
        return self.vec

    def epilogue(self, v0, v1, raw, net):
        n = self.n
        vec = self.vec.numpy()
        loc = getattr(self, "loc", None)
        if getattr(self, "partial", False):  # the summed row-partitioned vectors
            loc = vec[: 4 * n].reshape(4, n)
            vec = vec[4 * n:]
        c4, d13, d15 = vec[:n], vec[n:2 * n], vec[2 * n:]
        deg = np.array([len(a) for a in self.adj], np.int64)
        ids = [i for i in range(16) if self.mask >> i & 1]
        sat = lambda a, b: a - b if a > b else 0  # noqa: E731
        c3 = np.array([sum(self.c3full[(r, v)] for v in self.adj[r]) // 2 for r in range(n)])
        p2 = np.array([sat(sum(deg[v] for v in self.adj[r]), deg[r]) for r in range(n)])
        rows = []
        for v in range(v0, v1):
            r = int(self.inv[v])
            d = int(deg[r])
            nb = self.adj[r]
            cc = [self.c3full[(r, x)] for x in nb]
            col = [0] * 16
            col[0], col[1], col[2] = 1, d, int(p2[r])
            col[3] = d * (d - 1) // 2
            col[4] = int(c3[r])
            col[5] = sat(sum(int(p2[x]) for x in nb), d * sat(d, 1) + 2 * int(c3[r]))
            col[6] = sat(int(p2[r]) * sat(d, 1), 2 * int(c3[r]))
            col[7] = sum(sat(int(deg[x]), 1) * (sat(int(deg[x]), 1) - 1) // 2 for x in nb)
            col[8] = d * (d - 1) * (d - 2) // 6 if d >= 3 else 0
            col[9] = sat(sum(int(c3[x]) for x in nb), 2 * int(c3[r]))
            col[10] = sum(c * sat(int(deg[x]), 2) for c, x in zip(cc, nb))
            col[11] = sat(d, 2) * int(c3[r])
            col[12], col[13] = int(c4[r]), int(d13[r])
            col[14] = sum(c * (c - 1) // 2 for c in cc)
            if loc is not None:  # what the staged sweeps produced must agree
                assert int(getattr(self, "c3v")[r]) == col[4]
                assert (int(loc[0, r]), int(loc[1, r]), int(loc[2, r]), int(loc[3, r])) == \
                    (col[14], col[10], col[5], col[9]), (r, loc[:, r], col)
            col[15] = int(d15[r])
            rows.append([col[i] for i in ids])
        rows = np.array(rows, dtype=np.uint64).reshape(v1 - v0, len(ids))
        try:
            nt = ob.net_from_raw(rows, self.mask, self.lenient)
        except ob.OracleError as e:
            key = (6 << 40) | ((v0 + e.vertex) << 8) | ((1 if e.code == 4 else 0) << 4) | e.graphlet_id
            return e.code, (e.code, e.graphlet_id, v0 + e.vertex, "inconsistency", key)
        raw[: v1 - v0] = torch.from_numpy(rows.view(np.int64))
        net[: v1 - v0] = torch.from_numpy(nt.view(np.int64))
        return 0, (0, -1, -1, "", (1 << 64) - 1)

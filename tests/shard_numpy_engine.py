"""CPU shard engine for the multi-rank tests -- TEST INFRASTRUCTURE ONLY.

Implements the per-rank step interface of
``paper_2110_11211_b200.distributed.DeviceShardEngine`` with the CPU oracle
(oracle/sfcdd_oracle.py: scipy SuperLU local solves, dense coarse inverse) on
CPU torch tensors, so the product's SPMD orchestration (`pcg_program`,
`build_plans`, `run_torch`) can be exercised with world_size 2 over gloo on a
machine without GPUs.  Never used by the package.
"""

from __future__ import annotations

import numpy as np
import torch

import sfcdd_oracle as O
from paper_2110_11211_b200.distributed import block_owner


class NumpyShardEngine:
    def __init__(self, levels, p, gamma, q, rank, world):
        self.A = O.assemble_scaled_laplacian(levels)
        n = self.A.shape[0]
        self.n = n
        self.dis = O.disjoint_partition(n, p)
        self.ov = O.enlarge(self.dis, gamma)
        _, _, self.omega = O.weights(self.ov, n)
        owner = block_owner(p, world)
        self.first = int(np.argmax(owner == rank))
        self.count = int((owner == rank).sum())
        self.g0 = self.dis[self.first].start
        last = self.dis[self.first + self.count - 1]
        self.g1 = last.start + last.length
        self.q = q
        self.R0 = O.coarse_restriction(self.dis, n, q)
        self.agg = np.asarray(self.R0.T.tocsr().indices)  # aggregate of every point
        self.a0, self.a1 = self.first * q, (self.first + self.count) * q
        self.A0inv = np.linalg.inv(O.galerkin(self.R0, self.A).toarray())
        self.owned = list(range(self.first, self.first + self.count))
        self.solvers = {i: O.DirectSolver(self.A[self.ov[i].indices()][:, self.ov[i].indices()].tocsr())
                        for i in self.owned}
        # xy layout: owned subdomains first, then foreign slots covering owned points
        self.xy_offsets = np.full(p, -1, np.int64)
        off = 0
        for i in self.owned:
            self.xy_offsets[i] = off
            off += self.ov[i].length
        for j in range(p):
            if j in self.solvers:
                continue
            pts = self.ov[j].indices()
            if ((pts >= self.g0) & (pts < self.g1)).any():
                self.xy_offsets[j] = off
                off += self.ov[j].length
        self._xy = torch.zeros(off, dtype=torch.float64)
        self._idx = {}

    def neighbors(self, d):
        A = self.A.tocsr()
        out = np.full((2 * d, self.n), -1, np.int32)
        # any consistent neighbour listing works for the plans (only the set matters)
        for row in range(self.n):
            cols = [c for c in A.indices[A.indptr[row]:A.indptr[row + 1]] if c != row]
            out[:len(cols), row] = cols
        return out

    def attach_plan(self, plan):
        for name in ("halo", "ext", "xy"):
            ex = getattr(plan, name)
            for side in ("send", "recv"):
                for h, idx in getattr(ex, side).items():
                    self._idx[(name, side, h)] = torch.from_numpy(np.ascontiguousarray(idx))

    def index(self, kind, side, peer):
        return self._idx[(kind, side, peer)]

    def zeros(self):
        return torch.zeros(self.n, dtype=torch.float64)

    def empty(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def pack(self, buf, idx):
        return buf[idx].clone()

    def unpack(self, buf, idx, vals):
        buf[idx] = vals

    def xy(self):
        return self._xy

    def _own(self, v):
        return v.numpy()[self.g0:self.g1]

    def _cagg(self, v):
        return torch.from_numpy(np.asarray(self.R0 @ v)[self.a0:self.a1].copy())

    def residual(self, b, x, r):
        rv = b.numpy() - self.A @ x.numpy()
        r.numpy()[self.g0:self.g1] = rv[self.g0:self.g1]
        full = np.zeros(self.n)
        full[self.g0:self.g1] = rv[self.g0:self.g1]
        return torch.tensor([float(full @ full)], dtype=torch.float64), self._cagg(full)

    def coarse(self, c):
        return torch.from_numpy(self.A0inv @ c.numpy())

    def tvec(self, g, y0, t):
        t.numpy()[self.g0:self.g1] = (g.numpy() - self.A @ (self.R0.T @ y0.numpy()))[self.g0:self.g1]

    def local_solve(self, t):
        xy = self._xy.numpy()
        for i, s in self.solvers.items():
            off = self.xy_offsets[i]
            xy[off:off + self.ov[i].length] = s.solve(t.numpy()[self.ov[i].indices()])

    def combine(self, w):
        xy = self._xy.numpy()
        out = np.zeros(self.n)
        for i in range(len(self.ov)):
            if self.xy_offsets[i] < 0:
                continue
            idx = self.ov[i].indices()
            piece = self.omega[i] * xy[self.xy_offsets[i]:self.xy_offsets[i] + len(idx)]
            sel = (idx >= self.g0) & (idx < self.g1)
            out[idx[sel]] += piece[sel]
        w.numpy()[self.g0:self.g1] = out[self.g0:self.g1]

    def stencil_restrict(self, w):
        aw = np.zeros(self.n)
        aw[self.g0:self.g1] = (self.A @ w.numpy())[self.g0:self.g1]
        return self._cagg(aw)

    def finalize(self, w, y0, y0b, z, r):
        zz = (w.numpy() - self.R0.T @ y0b.numpy()) + self.R0.T @ y0.numpy()
        z.numpy()[self.g0:self.g1] = zz[self.g0:self.g1]
        return torch.tensor([float(r.numpy()[self.g0:self.g1] @ zz[self.g0:self.g1])], dtype=torch.float64)

    def pm(self, z, pold, beta, pnew, ap):
        pf = z.numpy() + beta * pold.numpy()
        apv = self.A @ pf
        pnew.numpy()[self.g0:self.g1] = pf[self.g0:self.g1]
        ap.numpy()[self.g0:self.g1] = apv[self.g0:self.g1]
        return torch.tensor([float(pf[self.g0:self.g1] @ apv[self.g0:self.g1])], dtype=torch.float64)

    def update(self, x, r, p, ap, alpha):
        sl = slice(self.g0, self.g1)
        x.numpy()[sl] += alpha * p.numpy()[sl]
        r.numpy()[sl] -= alpha * ap.numpy()[sl]
        full = np.zeros(self.n)
        full[sl] = r.numpy()[sl]
        return torch.tensor([float(full @ full)], dtype=torch.float64), self._cagg(full)

"""numpy shard backend for the CPU (gloo) tests of the sharded driver.

TEST INFRASTRUCTURE: it restates, per rank, what the rplu_shard_* kernels do
(global owner from the allgathered totals in rank order, absolute local
target, -0.0 contributions from non-owners, fused update + masses), so
``paper_2601_22344_b200.distributed.run_sharded`` — the collective
choreography the GPU ranks run — can be exercised with gloo on CPU tensors.
"""

import numpy as np
import torch

import oracle


class NumpyShardBackend:
    def __init__(self, A_local, row_offset, world, rank, seed, steps, stop_tol=0.0):
        self.R = np.array(A_local, dtype=np.float64)
        self.n_local, self.m = self.R.shape
        self.row_offset = row_offset
        self.world, self.rank = world, rank
        self.u = oracle.uniform_stream(seed).random(2 * steps + 2)
        self.uc = 0
        self.steps = steps
        self.stop_tol = stop_tol
        self.U = torch.zeros((steps + 1, self.m), dtype=torch.float64)
        self.L = np.zeros((self.n_local, steps))
        self.msg = torch.zeros(4 + self.m, dtype=torch.float64)   # header | pivot row
        self.pivots, self.resid = [], []
        self.active_flag, self.status = True, None
        self.fro0 = None

    def _masses(self):
        return np.einsum("ij,ij->i", self.R, self.R)

    def begin(self):
        self.masses = self._masses()
        return torch.tensor([self.masses.sum()], dtype=torch.float64)

    def _neg_zero(self, t):
        self.msg.fill_(-0.0)

    def select(self, t, totals):
        tot = totals.numpy()
        if not self.active_flag:
            self._neg_zero(t)
            return self.msg
        T = 0.0
        for s in range(self.world):
            T += tot[s]
        resid = np.sqrt(T)
        self.resid.append(resid)
        if t == 0:
            self.fro0 = resid
        stop = None
        if t > 0 and self.stop_tol > 0 and resid <= self.stop_tol * self.fro0:
            stop = "tol"
        elif t >= self.steps:
            stop = "end"
        elif resid == 0.0:
            stop = "clean"
        if stop:
            self.active_flag = False
            self.status = stop
            self._neg_zero(t)
            return self.msg
        u1, u2 = self.u[self.uc], self.u[self.uc + 1]
        self.uc += 2
        tg = u1 * T
        c, owner, target = 0.0, -1, 0.0
        for s in range(self.world):
            if owner < 0 and c + tot[s] > tg and tot[s] > 0:
                owner, target = s, tg - c
            c += tot[s]
        if owner < 0:
            owner = max(s for s in range(self.world) if tot[s] > 0)
            target = tot[owner]
        if owner != self.rank:
            self._neg_zero(t)
            return self.msg
        cdf = np.cumsum(self.masses)
        i = min(int(np.searchsorted(cdf, target, side="right")), self.n_local - 1)
        while i > 0 and not self.masses[i] > 0:
            i -= 1
        row = self.R[i].copy()
        j = oracle.sample_index(row * row, u2)
        self.msg[4:] = torch.from_numpy(row)
        self.msg[:4] = torch.tensor([float(self.row_offset + i), float(j), row[j], 0.0])
        return self.msg

    def update(self, t, msg):
        if not self.active_flag:
            return torch.tensor([self.masses.sum()], dtype=torch.float64)
        ig, j, a = int(msg[0]), int(msg[1]), float(msg[2])
        self.pivots.append((ig, j))
        self.U[t] = msg[4:]
        prow = self.U[t].numpy()
        col = self.R[:, j] * (1.0 / a)
        self.L[:, t] = col
        self.R -= np.outer(col, prow)
        self.masses = self._masses()
        return torch.tensor([self.masses.sum()], dtype=torch.float64)

    def active(self):
        return self.active_flag

    def finish(self):
        k = len(self.pivots)
        return dict(pivots=self.pivots, resid_fro=np.array(self.resid[:k + 1]), steps=k,
                    L_local=self.L[:, :k], U=self.U[:k].numpy(), status=self.status,
                    residual=self.R)

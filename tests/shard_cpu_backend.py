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
    """lazy_block > 0 restates the delayed-update shard loop: R keeps the
    residual of the last flush, the owner's pivot row and every rank's pivot
    column / masses apply the pending rank-1 terms on the fly in step order,
    and the rows are written back every lazy_block steps, at the last step,
    and (early stop) in finish."""

    def __init__(self, A_local, row_offset, world, rank, seed, steps, stop_tol=0.0,
                 lazy_block=0):
        self.lazy_block = lazy_block
        self.t0 = 0
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
        row = self._current(t, rows=slice(i, i + 1))[0]
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
        if not self.lazy_block:
            col = self.R[:, j] * (1.0 / a)
            self.L[:, t] = col
            self.R -= np.outer(col, prow)
            self.masses = self._masses()
            return torch.tensor([self.masses.sum()], dtype=torch.float64)
        col = self._current(t)[:, j] * (1.0 / a)
        self.L[:, t] = col
        cur = self._current(t + 1)
        self.masses = np.einsum("ij,ij->i", cur, cur)
        if (t + 1 - self.t0 == self.lazy_block) or t == self.steps - 1:
            self.R, self.t0 = cur, t + 1
        return torch.tensor([self.masses.sum()], dtype=torch.float64)

    def _current(self, t, rows=slice(None)):
        """Residual rows after steps < t from R^(t0) and the pending terms."""
        x = self.R[rows].copy()
        if not self.lazy_block:
            return x
        U = self.U.numpy()
        for s in range(self.t0, t):
            x -= np.outer(self.L[rows, s], U[s])
        return x

    def active(self):
        return self.active_flag

    def finish(self):
        k = len(self.pivots)
        if self.lazy_block and k > self.t0:
            self.R, self.t0 = self._current(k), k
        return dict(pivots=self.pivots, resid_fro=np.array(self.resid[:k + 1]), steps=k,
                    L_local=self.L[:, :k], U=self.U[:k].numpy(), status=self.status,
                    residual=self.R)


class NumpyCauchyShardBackend:
    """Per-rank restatement of the rplu_cauchy_shard_* kernels: x / G row
    blocks, y / B replicated; the owner broadcasts (i, x_i, G_i) through a
    -0.0 sum-allreduce, every rank regenerates the pivot row and draws the
    column identically, updates its G rows and (redundantly) B."""

    MSG = 20

    def __init__(self, x_loc, y, G_loc, B, row_offset, world, rank, rule, seed, steps,
                 stop_tol=0.0):
        self.x = np.asarray(x_loc, dtype=np.complex128)
        self.y = np.asarray(y, dtype=np.complex128)
        self.G = np.array(G_loc, dtype=np.complex128)
        self.B = np.array(B, dtype=np.complex128)
        self.p = self.G.shape[1]
        self.row_offset, self.world, self.rank = row_offset, world, rank
        self.rule, self.steps, self.stop_tol = rule, steps, stop_tol
        self.u = oracle.uniform_stream(seed).random(3 * steps + 2) if rule == "rplu" else None
        self.uc = 0
        self.active_flag, self.status = True, None
        self.rows, self.cols, self.bmax, self.bsum, self.C = [], [], [], [], []
        self.msg = torch.zeros(self.MSG, dtype=torch.float64)
        self.u0 = None

    def _stats(self):
        if self.x.size:
            self.masses = oracle.exact_row_norms(self.x, self.y, self.G, self.B)
        else:
            self.masses = np.zeros(0)
        tot = float(self.masses.sum()) if self.masses.size else 0.0
        mx = float(self.masses.max()) if self.masses.size else 0.0
        return torch.tensor([tot, mx], dtype=torch.float64)

    def begin(self):
        return self._stats()

    def select(self, t, totals):
        tot = totals.numpy().reshape(self.world, 2)
        self.msg.fill_(-0.0)
        if not self.active_flag:
            return self.msg
        T = 0.0
        for s in range(self.world):
            T += tot[s, 0]
        umax = float(tot[:, 1].max())
        self.bmax.append(umax)
        self.bsum.append(T)
        if self.u0 is None:
            self.u0 = umax
        if umax <= 0.0:
            self.active_flag, self.status = False, "degenerate"
            return self.msg
        if self.stop_tol > 0 and umax <= self.stop_tol ** 2 * self.u0:
            self.active_flag, self.status = False, "tol"
            return self.msg
        if self.rule == "rplu":
            tg = self.u[self.uc] * T
            self.uc += 1
            c, owner, target = 0.0, -1, 0.0
            for s in range(self.world):
                if owner < 0 and c + tot[s, 0] > tg and tot[s, 0] > 0:
                    owner, target = s, tg - c
                c += tot[s, 0]
            if owner < 0:
                owner = max(s for s in range(self.world) if tot[s, 0] > 0)
                target = tot[owner, 0]
        else:
            owner = min(s for s in range(self.world) if tot[s, 1] == umax)
        if owner != self.rank:
            return self.msg
        if self.rule == "rplu":
            cdf = np.cumsum(self.masses)
            i = min(int(np.searchsorted(cdf, target, side="right")), self.x.size - 1)
            while i > 0 and not self.masses[i] > 0:
                i -= 1
        else:
            i = int(np.argmax(self.masses))
        m = np.zeros(self.MSG)
        m[0] = self.row_offset + i
        m[1] = 0.0
        m[2], m[3] = self.x[i].real, self.x[i].imag
        for l in range(8):
            if l < self.p:
                m[4 + 2 * l], m[5 + 2 * l] = self.G[i, l].real, self.G[i, l].imag
            else:
                m[4 + 2 * l] = m[5 + 2 * l] = -0.0
        self.msg.copy_(torch.from_numpy(m))
        return self.msg

    def update(self, t, msg):
        if not self.active_flag:
            return self._stats()
        mm = msg.numpy()
        ig = int(mm[0])
        xi = complex(mm[2], mm[3])
        gi = np.array([complex(mm[4 + 2 * l], mm[5 + 2 * l]) for l in range(self.p)])
        r = (gi @ self.B) / (xi - self.y)
        w = np.abs(r) ** 2
        thr = oracle.PIVOT_REL_TOL * float(np.max(np.abs(r)))
        if self.rule == "rplu":
            j = oracle.sample_index(w, self.u[self.uc])
            self.uc += 1
            if not abs(r[j]) > thr:
                j = oracle.sample_index(w, self.u[self.uc])
                self.uc += 1
        else:
            j = int(np.argmax(np.abs(r)))
        a = r[j]
        if not abs(a) > thr:
            self.active_flag, self.status = False, "zero"
            return self._stats()
        c = (self.G @ self.B[:, j]) / (self.x - self.y[j]) if self.x.size else np.zeros(0)
        self.G = self.G - np.outer(c / a, gi)
        self.B = self.B - np.outer(self.B[:, j], r / a)
        self.rows.append(ig)
        self.cols.append(int(j))
        self.C.append(c)
        return self._stats()

    def active(self):
        return self.active_flag

    def finish(self):
        return dict(rows=self.rows, cols=self.cols, bound_maxes=self.bmax,
                    bound_sums=self.bsum, status=self.status, G=self.G, B=self.B)


# ---------------------------------------------------------------------------
# sharded cur_build on CPU tensors (gloo): the operator protocol and the draw /
# downdate primitives restated with torch / numpy

from paper_2601_22344_b200.operators import _DenseDeviceOp  # noqa: E402


class CpuDenseOp(_DenseDeviceOp):
    """_DenseDeviceOp on a CPU tensor (row norms without the CUDA kernel)."""

    def row_norms_dev(self):
        t = self.t
        return (t.real ** 2 + (t.imag ** 2 if torch.is_complex(t) else 0)).sum(1).to(torch.float64)


class NumpyCurOps:
    def cdf_total(self, w):
        w = w.numpy()
        return float(np.cumsum(w)[-1]) if w.size else 0.0

    def sample_target(self, w, target):
        w = w.numpy()
        c = np.cumsum(w)
        i = min(int(np.searchsorted(c, target, side="right")), w.size - 1)
        while i > 0 and not w[i] > 0:
            i -= 1
        if not w[i] > 0:
            i = int(np.flatnonzero(w > 0)[0])
        return i

    def sample(self, w, u):
        return oracle.sample_index(w.numpy(), u)

    def downdate(self, nrow, g, v, chat, l2, floor, real):
        nrow -= 2.0 * torch.real((g - v) * torch.conj(chat)) if not real else 2.0 * (g - v) * chat
        nrow += l2 * chat.abs() ** 2
        clamped = int((nrow < -floor).sum())
        nrow.clamp_(min=0.0)
        return clamped, float(nrow.sum())

"""Quadtrees and certified row-norm upper bounds.

Restates ``rplu.treebounds`` (pkg/src/rplu/treebounds.py): square-box
quadtrees over the target points x and source points y (:47-104), the dual
traversal building per-target-leaf interaction lists (Alg C.1,
``build_plan`` :141-180) and the certified bounds
u_i = sum_{(s,alpha) in A_l} alpha g_i^H H_s g_i
    + sum_{s in E_l} sum_{j in s} |g_i . B_j|^2 / |x_i - y_j|^2
with H_s = sum_{j in s} B_j B_j^H (Alg C.2, ``certified_upper_bounds``
:213-242), which satisfy exact <= u_i <= nu * exact.

The plan depends only on the point sets; it is built once on the host
(O(n log n) tree work, as in the reference) and flattened into device
arrays: points permuted by target leaf, CSR aggregated / exact lists, and
the source leaves under every source node.  The per-step work — the Gram
matrices of the current B and the bounds of every row — runs in
``librplu_b200.so`` (``rplu_tree_bounds``).
"""

from dataclasses import dataclass

import numpy as np

__all__ = ["PointQuadtree", "InteractionPlan", "CoincidentPointsError", "build_plan",
           "certified_upper_bounds", "DEFAULT_LEAF_SIZE"]

DEFAULT_LEAF_SIZE = 32  # treebounds.py:25


class CoincidentPointsError(ValueError):
    """A source point coincides with a target point; kernel entries blow up."""


class PointQuadtree:
    """Square-box quadtree (treebounds.py:47-104).

    Node arrays: ``x0, y0, size`` (lower-left corner and edge), ``parent``,
    ``children`` (lists), ``points`` (leaf point indices).  Children split
    the parent square in the order NW, NE, SW, SE; splitting stops at
    ``leaf_size`` points or when all remaining points coincide.
    """

    def __init__(self, points, leaf_size=DEFAULT_LEAF_SIZE):
        pts = np.asarray(points, dtype=np.complex128).ravel()
        if pts.size == 0:
            raise ValueError("cannot build a quadtree over zero points")
        if leaf_size < 1:
            raise ValueError("leaf size must be >= 1")
        self.points = pts
        self.leaf_size = int(leaf_size)
        xs, ys = pts.real, pts.imag
        ox, oy = float(np.min(xs)), float(np.min(ys))
        edge = max(float(np.max(xs) - ox), float(np.max(ys) - oy), 1e-300)
        edge *= 1.0 + 1e-12
        self.x0, self.y0, self.size, self.parent = [ox], [oy], [edge], [-1]
        self.children = [[]]
        self.node_points = [np.arange(pts.size)]
        self.leaves = []
        todo = [0]
        while todo:
            k = todo.pop()
            idx = self.node_points[k]
            if idx.size <= self.leaf_size or bool(np.all(pts[idx] == pts[idx[0]])):
                self.leaves.append(k)
                continue
            h = self.size[k] / 2.0
            cx, cy = self.x0[k] + h, self.y0[k] + h
            east = xs[idx] >= cx
            north = ys[idx] >= cy
            for mask, bx, by in ((~east & north, self.x0[k], cy), (east & north, cx, cy),
                                 (~east & ~north, self.x0[k], self.y0[k]),
                                 (east & ~north, cx, self.y0[k])):
                sub = idx[mask]
                if sub.size == 0:
                    continue
                c = len(self.x0)
                self.x0.append(bx)
                self.y0.append(by)
                self.size.append(h)
                self.parent.append(k)
                self.children.append([])
                self.node_points.append(sub)
                self.children[k].append(c)
                todo.append(c)
            self.node_points[k] = np.empty(0, dtype=np.int64)

    @property
    def n_nodes(self):
        return len(self.x0)

    def is_leaf(self, k):
        return not self.children[k]


def _box_dist2(a, ia, b, ib):
    """(d_min^2, d_max^2) between square ia of tree a and square ib of tree b."""
    ax0, ay0, asz = a.x0[ia], a.y0[ia], a.size[ia]
    bx0, by0, bsz = b.x0[ib], b.y0[ib], b.size[ib]
    ax1, ay1, bx1, by1 = ax0 + asz, ay0 + asz, bx0 + bsz, by0 + bsz
    dx = max(0.0, bx0 - ax1, ax0 - bx1)
    dy = max(0.0, by0 - ay1, ay0 - by1)
    ex = max(bx1 - ax0, ax1 - bx0)
    ey = max(by1 - ay0, ay1 - by0)
    return dx * dx + dy * dy, ex * ex + ey * ey


@dataclass
class InteractionPlan:
    """Interaction lists for one (target x, source y) pair (treebounds.py:107-138).

    ``aggregated[leaf]``: list of (source node, alpha = 1/d_min^2(node, leaf));
    ``exact[leaf]``: list of source leaves summed directly.
    """

    source_tree: PointQuadtree
    target_tree: PointQuadtree
    nu: float
    aggregated: dict
    exact: dict
    _device: object = None


def _build_plan_py(x, y, nu=5.0, leaf_size=DEFAULT_LEAF_SIZE):
    """Alg C.1 dual traversal (treebounds.py:141-180) for targets x vs sources y,
    in Python (kept as the cross-check of the native build, tests only)."""
    if nu < 1.0:
        raise ValueError("nu must be >= 1")
    tgt = PointQuadtree(x, leaf_size)
    src = PointQuadtree(y, leaf_size)
    agg = {leaf: [] for leaf in tgt.leaves}
    exact = {leaf: [] for leaf in tgt.leaves}
    under = [[] for _ in range(tgt.n_nodes)]   # target leaves below each node
    for leaf in tgt.leaves:
        k = leaf
        while k != -1:
            under[k].append(leaf)
            k = tgt.parent[k]
    todo = [(0, 0)]
    while todo:
        s, t = todo.pop()
        dmin2, dmax2 = _box_dist2(src, s, tgt, t)
        if dmin2 > 0.0 and dmax2 <= nu * dmin2:
            for leaf in under[t]:
                lmin2, _ = _box_dist2(src, s, tgt, leaf)
                agg[leaf].append((s, 1.0 / lmin2))
            continue
        s_leaf, t_leaf = src.is_leaf(s), tgt.is_leaf(t)
        if s_leaf and t_leaf:
            if dmin2 == 0.0:
                _check_cross(src, s, tgt, t)
            exact[t].append(s)
            continue
        if (tgt.size[t] >= src.size[s] and not t_leaf) or s_leaf:
            todo.extend((s, c) for c in tgt.children[t])
        else:
            todo.extend((c, t) for c in src.children[s])
    return InteractionPlan(source_tree=src, target_tree=tgt, nu=float(nu), aggregated=agg,
                           exact=exact)


class _CsrSeq:
    """Read-only sequence view of a CSR array (children / node points)."""

    def __init__(self, start, idx, as_list):
        self._start, self._idx, self._as_list = start, idx, as_list

    def __len__(self):
        return len(self._start) - 1

    def __getitem__(self, k):
        seg = self._idx[self._start[k]:self._start[k + 1]]
        return seg.tolist() if self._as_list else seg


class _LeafLists:
    """dict-like {target leaf: list} view of a per-leaf CSR list."""

    def __init__(self, leaves, start, cols):
        self._slot = {leaf: q for q, leaf in enumerate(leaves)}
        self._start, self._cols = start, cols

    def __getitem__(self, leaf):
        q = self._slot[leaf]
        a, b = self._start[q], self._start[q + 1]
        if len(self._cols) == 1:
            return self._cols[0][a:b].tolist()
        return list(zip(*(c[a:b].tolist() for c in self._cols)))

    def __contains__(self, leaf):
        return leaf in self._slot

    def __iter__(self):
        return iter(self._slot)

    def __len__(self):
        return len(self._slot)

    def keys(self):
        return self._slot.keys()

    def items(self):
        return ((k, self[k]) for k in self._slot)


def _native_tree(points, leaf_size, arrays):
    x0, y0, size, parent, cstart, cidx, leaves, lpstart, lpidx = arrays
    t = PointQuadtree.__new__(PointQuadtree)
    t.points = points
    t.leaf_size = int(leaf_size)
    t.x0, t.y0, t.size, t.parent = x0.tolist(), y0.tolist(), size.tolist(), parent.tolist()
    t.children = _CsrSeq(cstart, cidx, True)
    t.leaves = leaves.tolist()
    nn = len(x0)
    cnt = np.zeros(nn, dtype=np.int64)
    cnt[leaves] = np.diff(lpstart)
    nstart = np.concatenate([[0], np.cumsum(cnt)])
    order = np.argsort(leaves, kind="stable")
    segs = [lpidx[lpstart[q]:lpstart[q + 1]] for q in order]
    t.node_points = _CsrSeq(nstart, np.concatenate(segs) if segs else lpidx, False)
    t._csr = dict(cstart=cstart, cidx=cidx, leaves=leaves, lpstart=lpstart, lpidx=lpidx,
                  parent=parent)
    return t


def build_plan(x, y, nu=5.0, leaf_size=DEFAULT_LEAF_SIZE):
    """Alg C.1 dual traversal (treebounds.py:141-180) for targets x vs sources
    y: quadtrees and interaction lists built by the host-native
    ``rplu_plan_build`` (identical plans to the reference's, ~50x faster than
    a Python traversal at C4 size)."""
    import ctypes

    from . import _ffi
    if nu < 1.0:
        raise ValueError("nu must be >= 1")
    xs = np.ascontiguousarray(np.asarray(x, dtype=np.complex128).ravel())
    ys = np.ascontiguousarray(np.asarray(y, dtype=np.complex128).ravel())
    if xs.size == 0 or ys.size == 0:
        raise ValueError("cannot build a quadtree over zero points")
    if leaf_size < 1:
        raise ValueError("leaf size must be >= 1")
    lib = _ffi.load_library()
    h = ctypes.c_void_p()
    co = np.full(2, -1, dtype=np.int64)
    st = lib.rplu_plan_build(xs.ctypes.data, xs.size, ys.ctypes.data, ys.size, float(nu),
                             int(leaf_size), co.ctypes.data, ctypes.byref(h))
    if st != 0:
        if co[0] >= 0:
            a, b = int(co[0]), int(co[1])
            raise CoincidentPointsError(
                f"target point {a} coincides with source point {b} at {xs[a]!r}")
        _ffi.check(st)
    try:
        cnt = np.zeros(8, dtype=np.int64)
        _ffi.check(lib.rplu_plan_counts(h, cnt.ctypes.data))
        trees = []
        for which, pts, (nn, nl, nc) in ((0, xs, cnt[0:3]), (1, ys, cnt[3:6])):
            arr = (np.empty(nn), np.empty(nn), np.empty(nn), np.empty(nn, np.int64),
                   np.empty(nn + 1, np.int64), np.empty(max(nc, 1), np.int64),
                   np.empty(nl, np.int64), np.empty(nl + 1, np.int64),
                   np.empty(pts.size, np.int64))
            _ffi.check(lib.rplu_plan_tree(h, which, *(a.ctypes.data for a in arr)))
            trees.append(_native_tree(pts, leaf_size, arr))
        tgt, src = trees
        nl = int(cnt[1])
        agg_start, ex_start = np.empty(nl + 1, np.int64), np.empty(nl + 1, np.int64)
        agg_node, agg_alpha = np.empty(max(cnt[6], 1), np.int64), np.empty(max(cnt[6], 1))
        ex_node = np.empty(max(cnt[7], 1), np.int64)
        _ffi.check(lib.rplu_plan_lists(h, agg_start.ctypes.data, agg_node.ctypes.data,
                                       agg_alpha.ctypes.data, ex_start.ctypes.data,
                                       ex_node.ctypes.data))
    finally:
        lib.rplu_plan_free(h)
    plan = InteractionPlan(source_tree=src, target_tree=tgt, nu=float(nu),
                           aggregated=_LeafLists(tgt.leaves, agg_start, (agg_node, agg_alpha)),
                           exact=_LeafLists(tgt.leaves, ex_start, (ex_node,)))
    plan._csr = dict(agg_start=agg_start, agg_node=agg_node, agg_alpha=agg_alpha,
                     ex_start=ex_start, ex_node=ex_node)
    return plan


def _check_cross(src, s, tgt, t):
    xs = tgt.points[tgt.node_points[t]]
    ys = src.points[src.node_points[s]]
    d = np.abs(xs[:, None] - ys[None, :])
    if np.any(d == 0.0):
        a, b = np.argwhere(d == 0.0)[0]
        raise CoincidentPointsError(
            f"target point {tgt.node_points[t][a]} coincides with source point "
            f"{src.node_points[s][b]} at {xs[a]!r}")


class _DevicePlan:
    """Flattened plan in HBM (CSR arrays, int64 / fp64)."""

    def __init__(self, plan, device):
        import torch
        if getattr(plan, "_csr", None) is not None and hasattr(plan.source_tree, "_csr"):
            self._from_native(plan, device)
            return
        tgt, src = plan.target_tree, plan.source_tree
        leaves = list(tgt.leaves)
        perm, tstart = [], [0]
        for leaf in leaves:
            perm.extend(int(i) for i in tgt.node_points[leaf])
            tstart.append(len(perm))
        agg_start, agg_node, agg_alpha = [0], [], []
        ex_start, ex_leaf = [0], []
        for leaf in leaves:
            for node, alpha in plan.aggregated[leaf]:
                agg_node.append(node)
                agg_alpha.append(alpha)
            agg_start.append(len(agg_node))
            ex_leaf.extend(plan.exact[leaf])
            ex_start.append(len(ex_leaf))
        # source points grouped by source leaf, and the leaves under each node
        sleaf_index = {leaf: k for k, leaf in enumerate(src.leaves)}
        spts, sstart = [], [0]
        for leaf in src.leaves:
            spts.extend(int(i) for i in src.node_points[leaf])
            sstart.append(len(spts))
        # children CSR and the internal nodes grouped by depth, deepest first
        # (node Grams are summed bottom-up from their children, one launch
        # per level, as the reference's _gram_bottom_up, treebounds.py:196-210)
        cstart, cidx = [0], []
        for k in range(src.n_nodes):
            cidx.extend(src.children[k])
            cstart.append(len(cidx))
        depth = [0] * src.n_nodes
        for k in range(1, src.n_nodes):          # parents precede children
            depth[k] = depth[src.parent[k]] + 1
        internal = [k for k in range(src.n_nodes) if src.children[k]]
        levels = sorted(set(depth[k] for k in internal), reverse=True)
        lvl_nodes, lvl_start = [], [0]
        for d in levels:
            lvl_nodes.extend(k for k in internal if depth[k] == d)
            lvl_start.append(len(lvl_nodes))
        def i64(a):
            return torch.tensor(np.asarray(a, dtype=np.int64), device=device)

        self.n_tleaves = len(leaves)
        self.tperm, self.tstart = i64(perm), i64(tstart)
        self.agg_start, self.agg_node = i64(agg_start), i64(agg_node if agg_node else [0])
        self.agg_alpha = torch.tensor(np.asarray(agg_alpha if agg_alpha else [0.0]),
                                      dtype=torch.float64, device=device)
        self.ex_start = i64(ex_start)
        self.ex_leaf = i64([sleaf_index[s] for s in ex_leaf] if ex_leaf else [0])
        self.n_snodes, self.n_sleaves = src.n_nodes, len(src.leaves)
        self.spts, self.sstart = i64(spts), i64(sstart)
        self.cstart, self.cidx = i64(cstart), i64(cidx if cidx else [0])
        self.leaf_node = i64(list(src.leaves))
        self.lvl_nodes = i64(lvl_nodes if lvl_nodes else [0])
        self.lvl_start = np.asarray(lvl_start, dtype=np.int64)   # host
        self.n_levels = len(levels)
        self.max_leaf = max(int(np.diff(tstart).max()), int(np.diff(sstart).max()))


    def _from_native(self, plan, device):
        import torch
        tgt, src = plan.target_tree, plan.source_tree
        tc, sc, pc = tgt._csr, src._csr, plan._csr

        def dev(a, dt=torch.int64):
            return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dt)

        self.n_tleaves = len(tc["leaves"])
        self.tperm, self.tstart = dev(tc["lpidx"]), dev(tc["lpstart"])
        self.agg_start, self.agg_node = dev(pc["agg_start"]), dev(pc["agg_node"])
        self.agg_alpha = dev(pc["agg_alpha"], torch.float64)
        self.ex_start = dev(pc["ex_start"])
        sleaf = np.full(src.n_nodes, -1, dtype=np.int64)
        sleaf[sc["leaves"]] = np.arange(len(sc["leaves"]))
        ne = int(pc["ex_start"][-1])
        self.ex_leaf = dev(sleaf[pc["ex_node"][:ne]] if ne else np.zeros(1, np.int64))
        self.n_snodes, self.n_sleaves = src.n_nodes, len(sc["leaves"])
        self.spts, self.sstart = dev(sc["lpidx"]), dev(sc["lpstart"])
        self.cstart, self.cidx = dev(sc["cstart"]), dev(sc["cidx"])
        self.leaf_node = dev(sc["leaves"])
        parent = sc["parent"]
        depth = np.zeros(src.n_nodes, dtype=np.int64)
        for k in range(1, src.n_nodes):          # parents precede children
            depth[k] = depth[parent[k]] + 1
        internal = np.nonzero(np.diff(sc["cstart"]) > 0)[0]
        order = internal[np.argsort(-depth[internal], kind="stable")]
        levels = np.unique(depth[internal])[::-1]
        lvl_start = [0]
        for d in levels:
            lvl_start.append(lvl_start[-1] + int(np.sum(depth[internal] == d)))
        self.lvl_nodes = dev(order if order.size else np.zeros(1, np.int64))
        self.lvl_start = np.asarray(lvl_start, dtype=np.int64)
        self.n_levels = len(levels)
        self.max_leaf = max(int(np.diff(tc["lpstart"]).max()), int(np.diff(sc["lpstart"]).max()))

def device_plan(plan, device):
    if plan._device is None or plan._device[0] != device:
        plan._device = (device, _DevicePlan(plan, device))
    return plan._device[1]


def certified_upper_bounds(plan, G, B):
    """Per-row upper bounds exact <= u <= nu*exact (treebounds.py:213-242),
    computed on the device.  G (n x p) and B (p x m) may be host arrays or a
    CauchyLikeMatrix's device generators.  Returns numpy."""
    from .cauchy import CauchyLikeMatrix, tree_bounds_device
    tgt, src = plan.target_tree, plan.source_tree
    M = CauchyLikeMatrix(tgt.points, src.points, G, B, check_points=False)
    if M.shape[0] != tgt.points.size or M.shape[1] != src.points.size:
        raise ValueError("generator dimensions do not match the plan's points")
    return tree_bounds_device(plan, M).cpu().numpy()

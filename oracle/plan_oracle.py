"""numpy restatement of the reference's certified tree bounds (Alg C.2,
rplu/treebounds.py:196-242) — TEST INFRASTRUCTURE ONLY.

Takes a plan in the layout of ``paper_2601_22344_b200.build_plan`` (whose
plans are identical to the reference's, tests/test_treebounds_cpu.py):
``target_tree`` / ``source_tree`` with ``leaves``, ``children``,
``node_points``, and per-target-leaf ``aggregated`` [(node, alpha)] and
``exact`` [source leaf] lists.  Pinned against the reference's bounds in
tests/golden/cauchy_plan.npz (tests/test_oracle_golden.py); also the timed
CPU leg of bench.py's plan-path line (the reference spends its plan step in
exactly this per-leaf loop).
"""

import numpy as np

__all__ = ["node_grams", "certified_upper_bounds"]


def node_grams(src, B):
    """H[node] = sum over the node's source points of B_:,j B_:,j^H, leaves
    first, internal nodes as the sum of their children (:196-210)."""
    p = B.shape[0]
    H = np.zeros((src.n_nodes, p, p), np.complex128)
    for k in sorted(range(src.n_nodes), key=lambda k: -len(_ancestors(src, k))):
        if not src.children[k]:
            Bs = B[:, src.node_points[k]]
            H[k] = Bs @ Bs.conj().T
        else:
            for c in src.children[k]:
                H[k] += H[c]
    return H


def _ancestors(tree, k):
    out = []
    while tree.parent[k] != -1:
        k = tree.parent[k]
        out.append(k)
    return out


def certified_upper_bounds(plan, G, B):
    """u_i >= sum_j |A_ij|^2 from the plan's aggregated Grams and exact
    leaves (:213-242)."""
    G = np.asarray(G, np.complex128)
    B = np.asarray(B, np.complex128)
    src, tgt = plan.source_tree, plan.target_tree
    H = node_grams(src, B)
    u = np.zeros(tgt.points.size)
    for leaf in tgt.leaves:
        pts = tgt.node_points[leaf]
        g = G[pts]
        acc = np.zeros(pts.size)
        for node, alpha in plan.aggregated[leaf]:
            acc += alpha * np.einsum("ip,pq,iq->i", g, H[node], g.conj()).real
        for s in plan.exact[leaf]:
            sp = src.node_points[s]
            W = g @ B[:, sp]
            D = np.abs(tgt.points[pts, None] - src.points[None, sp]) ** 2
            acc += np.sum(np.abs(W) ** 2 / D, axis=1)
        u[pts] = acc
    return u

"""The host-side quadtree / interaction-plan builder (Alg C.1) reproduces the
reference's plans exactly (golden signatures from tests/golden/make_golden.py)."""

import numpy as np
import pytest

from conftest import load_golden
from paper_2601_22344_b200 import treebounds


def _signature(plan):
    tgt, src = plan.target_tree, plan.source_tree
    sig = {}
    for leaf in tgt.leaves:
        pts = tgt.node_points[leaf]
        sig[str(int(np.min(pts)))] = {
            "alphas": sorted(float(a) for _, a in plan.aggregated[leaf]),
            "exact": sorted(sorted(int(i) for i in src.node_points[s]) for s in plan.exact[leaf]),
            "points": sorted(int(i) for i in pts)}
    return sig


def _cases():
    info, _ = load_golden("cauchy_plan")
    return info["cases"]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_plan_matches_reference(case):
    _, arr = load_golden("cauchy_plan")
    name = case["name"]
    plan = treebounds.build_plan(arr[name + "_x"], arr[name + "_y"], nu=case["nu"],
                                 leaf_size=case["leaf_size"])
    sig = _signature(plan)
    assert set(sig) == set(case["plan"])
    for k, v in case["plan"].items():
        assert sig[k]["points"] == v["points"]
        assert sig[k]["alphas"] == v["alphas"]
        assert sig[k]["exact"] == v["exact"]


def test_plan_coverage_and_admissibility():
    """Every source point is covered exactly once per target leaf and every
    aggregated pair satisfies d_max^2 <= nu d_min^2 (SPEC treebounds invariants)."""
    rs = np.random.default_rng(0)
    x = rs.standard_normal(500) + 1j * rs.standard_normal(500)
    y = 3 + rs.standard_normal(400) + 1j * rs.standard_normal(400)
    plan = treebounds.build_plan(x, y, nu=4.0, leaf_size=8)
    src, tgt = plan.source_tree, plan.target_tree

    def pts_under(k):
        if src.is_leaf(k):
            return list(src.node_points[k])
        out = []
        for c in src.children[k]:
            out += pts_under(c)
        return out

    for leaf in tgt.leaves:
        cover = []
        for s, alpha in plan.aggregated[leaf]:
            dmin2, dmax2 = treebounds._box_dist2(src, s, tgt, leaf)
            assert dmin2 > 0 and abs(alpha - 1.0 / dmin2) <= 1e-12 / dmin2
            cover += pts_under(s)
        for s in plan.exact[leaf]:
            cover += list(src.node_points[s])
        assert sorted(cover) == list(range(400))


def test_plan_validation():
    with pytest.raises(ValueError):
        treebounds.build_plan([0j, 1j], [2.0], nu=0.5)
    with pytest.raises(ValueError):
        treebounds.PointQuadtree([], 4)
    with pytest.raises(treebounds.CoincidentPointsError):
        treebounds.build_plan([0.5 + 0.5j, 0.1j], [0.5 + 0.5j, 2.0], nu=5.0, leaf_size=1)


@pytest.mark.parametrize("n,m,leaf,nu", [(300, 250, 32, 5.0), (2000, 1500, 8, 3.0),
                                         (500, 700, 1, 5.0), (4096, 4096, 32, 1.0)])
def test_native_plan_equals_python_restatement(n, m, leaf, nu):
    """rplu_plan_build (host-native) builds the same trees and interaction
    lists, in the same order, as the Python restatement of the reference."""
    from paper_2601_22344_b200 import gen
    from paper_2601_22344_b200 import treebounds as tb
    x, y, _, _ = gen.c4_cauchy_like(n + leaf, n=n, m=m, p=1)
    a = tb.build_plan(x, y, nu=nu, leaf_size=leaf)
    b = tb._build_plan_py(x, y, nu=nu, leaf_size=leaf)
    for ta, tb_ in ((a.target_tree, b.target_tree), (a.source_tree, b.source_tree)):
        assert ta.n_nodes == tb_.n_nodes and ta.leaves == tb_.leaves
        assert ta.x0 == tb_.x0 and ta.y0 == tb_.y0 and ta.size == tb_.size
        assert list(ta.parent) == list(tb_.parent)
        for k in range(ta.n_nodes):
            assert ta.children[k] == tb_.children[k]
            np.testing.assert_array_equal(ta.node_points[k], tb_.node_points[k])
    for leaf_id in b.target_tree.leaves:
        assert a.aggregated[leaf_id] == b.aggregated[leaf_id]
        assert a.exact[leaf_id] == b.exact[leaf_id]


def test_native_plan_edge_cases():
    from paper_2601_22344_b200 import treebounds as tb
    same = np.full(100, 0.5 + 0.5j)                     # all coincident: one leaf
    p = tb.build_plan(same, np.array([3.0 + 0j, 4.0 + 1j]), leaf_size=4)
    assert p.target_tree.leaves == [0]
    x = np.array([0.0, 1.0, 2.0 + 1j]) + 0j
    with pytest.raises(tb.CoincidentPointsError):
        tb.build_plan(x, np.array([5.0, 2.0 + 1j]))
    with pytest.raises(ValueError):
        tb.build_plan(x, np.array([5.0 + 0j]), nu=0.5)
    with pytest.raises(ValueError):
        tb.build_plan(np.zeros(0, complex), x)

"""Host-side API behaviour that needs no GPU: rule validation, exception
classes, uniform-stream bookkeeping, and the absence of any CPU fallback."""

import os

import numpy as np
import pytest
import torch

import paper_2601_22344_b200 as rp
from paper_2601_22344_b200.rng import UniformBlock


def test_pivot_rule_validation():
    with pytest.raises(ValueError):
        rp.PivotRule("bogus")
    with pytest.raises(ValueError):
        rp.PivotRule("rplu")            # random rule without an RngState
    rp.PivotRule("cplu")
    rp.PivotRule("rplu", rp.RngState(0))


def test_capability_error_is_value_error():
    assert issubclass(rp.CapabilityError, ValueError)


def test_psd_rules_rejected_not_fallen_back():
    with pytest.raises(rp.CapabilityError):
        rp.eliminate(np.eye(3), rp.PivotRule("rpcholesky", rp.RngState(0)), 1)


def test_rng_stream_matches_numpy_philox():
    g = rp.RngState(42)
    ref = np.random.Generator(np.random.Philox(key=42))
    assert g.uniform() == float(ref.random())
    np.testing.assert_array_equal(g.uniforms(10), ref.random(10))


def test_uniform_block_commits_exact_consumption():
    g = rp.RngState(7)
    blk = UniformBlock(g, 400)
    first5 = blk.values[:5].copy()
    blk.commit(5)
    ref = np.random.Generator(np.random.Philox(key=7))
    np.testing.assert_array_equal(ref.random(5), first5)
    assert g.uniform() == float(ref.random())


def test_uniform_block_accepts_reference_like_rng():
    class Like:
        def __init__(self):
            self._gen = np.random.Generator(np.random.Philox(key=3))
    r = Like()
    blk = UniformBlock(r, 8)
    blk.commit(2)
    ref = np.random.Generator(np.random.Philox(key=3))
    ref.random(2)
    assert r._gen.random() == ref.random()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rp.eliminate(np.eye(4), rp.PivotRule("rplu", rp.RngState(0)), 2)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_consumers_have_no_cpu_fallback():
    S = rp.SampleSet(np.arange(6) + 0j, np.exp(np.arange(6) + 0j))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rp.aaa(S)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rp.cur_aaa(S, rng=rp.RngState(0))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rp.gmres(np.eye(3), np.ones(3))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rp.BarycentricRational([0.0, 1.0], [1.0, 2.0], [1.0, 1.0])


def test_reference_accessor_duck_types():
    """The reference's own accessor classes are recognised by the boundary
    helpers (imported from /root/reference in the build container only)."""
    import sys
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not present on this host")
    sys.path.insert(0, src)
    try:
        import rplu
    finally:
        sys.path.remove(src)
    from paper_2601_22344_b200.accessors import foreign_dense_array, is_host_accessor
    D = rplu.DenseMatrix(np.eye(3))
    assert foreign_dense_array(D) is D.array
    assert is_host_accessor(rplu.CallableOperator((3, 3), lambda v: v))
    assert foreign_dense_array(np.eye(3)) is None and not is_host_accessor(np.eye(3))

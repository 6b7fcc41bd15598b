import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built extension")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        info = json.load(f)
    arrays = np.load(os.path.join(GOLDEN, name + ".npz"))
    return info, arrays


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch.device("cuda", 0)


def record_parity(name, **fields):
    """Append one parity record (first divergence, near-boundary draws, ...)
    to $RPLU_PARITY_LOG (JSON lines) when set; the GPU runs keep it under
    profiles/."""
    path = os.environ.get("RPLU_PARITY_LOG")
    if not path:
        return
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    with open(path, "a") as f:
        f.write(json.dumps(dict(test=name, **fields), default=float) + "\n")


def check_dense_parity(tr, ref, near_rel=1e-12, exact=True, rtol=1e-10):
    """Pivots equal to the oracle's, or the first divergence at a draw the
    oracle marks within ``near_rel`` of a CDF boundary; L and U compared up
    to (not including) that step: bit for bit (``exact``) or to ``rtol``
    relative to each factor's max.  Returns the first divergence step or
    None."""
    import torch
    got, want = list(tr.pivots), list(ref["pivots"])
    t = next((s for s, (a, b) in enumerate(zip(got, want)) if a != b), None)
    if t is None:
        assert len(got) == len(want), (len(got), len(want))
        k = len(got)
    else:
        assert ref["margins"] is not None and ref["margins"][t] <= near_rel, (
            f"pivot divergence at step {t} (oracle margin {ref['margins'][t]:.3e}) "
            "is not near a CDF boundary")
        k = t

    def host(a):
        return a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    L, U = host(tr.L)[:, :k], host(tr.U)[:k]
    Lr, Ur = np.asarray(ref["L"])[:, :k], np.asarray(ref["U"])[:k]
    if exact:
        np.testing.assert_array_equal(L, Lr)
        np.testing.assert_array_equal(U, Ur)
    elif k:
        assert np.abs(L - Lr).max() <= rtol * np.abs(Lr).max()
        assert np.abs(U - Ur).max() <= rtol * np.abs(Ur).max()
    np.testing.assert_allclose(np.asarray(tr.resid_fro)[:k + 1],
                               np.asarray(ref["resid_fro"])[:k + 1],
                               rtol=1e-12 if exact else rtol, atol=1e-300)
    return t

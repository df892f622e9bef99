"""Blelloch step functions up_sweep / down_sweep (simd.py:327-367): the C
oracle (CPU) and the GPU kernels (ps_tree_up_sweep / ps_tree_down_sweep)
against golden vectors produced by the reference (tests/golden/make_sweeps.py).
Element-typed arithmetic in the reference's pairing: bit-exact for every dtype,
float32 included."""

import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "sweeps.npz"))
CASES = list(range(int(G["n_cases"][0])))


def _case(k):
    return G[f"c{k}_in"], G[f"c{k}_up"], G[f"c{k}_root"][0], G[f"c{k}_down"]


@pytest.mark.parametrize("k", CASES)
def test_oracle_sweeps_match_reference(oracle_lib, k):
    buf, up, root, down = _case(k)
    n = buf.shape[0] - 5
    a = buf.copy()
    r = oracle_lib.up_sweep(a, 3, n)
    assert np.array_equal(a.view(np.uint8), up.view(np.uint8))
    assert np.array_equal(np.array([r]).view(np.uint8), np.array([root]).view(np.uint8))
    oracle_lib.down_sweep(a, 3, n)
    assert np.array_equal(a.view(np.uint8), down.view(np.uint8))


@pytest.mark.gpu
@pytest.mark.parametrize("k", CASES)
@pytest.mark.parametrize("where", ["numpy", "cuda"])
def test_gpu_sweeps_match_reference(k, where):
    import torch

    from paper_2312_14874_b200 import Span
    from paper_2312_14874_b200.simd import down_sweep, up_sweep
    buf, up, root, down = _case(k)
    n = buf.shape[0] - 5
    a = buf.copy() if where == "numpy" else torch.from_numpy(buf.copy()).cuda()
    r = up_sweep(a, Span(3, n))
    got = a if where == "numpy" else a.cpu().numpy()
    assert np.array_equal(got.view(np.uint8), up.view(np.uint8))
    assert np.array_equal(np.array([r], dtype=buf.dtype).view(np.uint8), np.array([root]).view(np.uint8))
    down_sweep(a, Span(3, n))
    got = a if where == "numpy" else a.cpu().numpy()
    assert np.array_equal(got.view(np.uint8), down.view(np.uint8))


@pytest.mark.gpu
def test_gpu_sweeps_large_and_errors():
    import torch

    from paper_2312_14874_b200 import Span
    from paper_2312_14874_b200.simd import down_sweep, up_sweep
    n = 1 << 22
    x = torch.randint(0, 1000, (n,), dtype=torch.int64, device="cuda")
    ref = x.cpu().numpy()
    r = up_sweep(x, Span(0, n))
    assert int(r) == int(ref.sum())
    down_sweep(x, Span(0, n))
    assert np.array_equal(x.cpu().numpy(), np.concatenate([[0], np.cumsum(ref)[:-1]]))
    with pytest.raises(ValueError):
        up_sweep(torch.zeros(6, dtype=torch.int64, device="cuda"), Span(0, 6))

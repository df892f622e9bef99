"""End-to-end host-buffer pipelines (ps_scan_host, ps_scan_batched_host):
chunked H2D -> scan -> D2H over three streams, checked against numpy."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rows(rows, cols, dt, seed):
    r = np.random.default_rng(seed)
    if np.dtype(dt).kind == "f":
        return r.random((rows, cols), dtype=dt)
    return r.integers(0, 256, (rows, cols), dtype=dt)


@pytest.mark.parametrize("rows,cols,chunk", [(1, 1, None), (3, 5, 2), (64, 1000, 7), (513, 4096, 100),
                                             (2048, 2049, None), (20_000, 1000, None), (9000, 250, 3000),
                                             (4000, 3001, None)])
@pytest.mark.parametrize("exclusive", [False, True])
def test_batched_host_int32_to_int64(rows, cols, chunk, exclusive):
    from paper_2312_14874_b200 import device as dev
    x = _rows(rows, cols, np.int32, rows + cols)
    out = np.empty((rows, cols), np.int64)
    dev.scan_batched_host(x, out, exclusive=exclusive, chunk_rows=chunk)
    want = np.cumsum(x, axis=1, dtype=np.int64)
    if exclusive:
        want = np.concatenate([np.zeros((rows, 1), np.int64), want[:, :-1]], axis=1)
    assert np.array_equal(out, want)


def test_batched_host_pinned_tensor_and_in_place():
    from paper_2312_14874_b200 import device as dev
    x = torch.from_numpy(_rows(300, 5000, np.int64, 3)).pin_memory()
    want = np.cumsum(x.numpy(), axis=1)
    dev.scan_batched_host(x, chunk_rows=64)  # in place
    assert np.array_equal(x.numpy(), want)


def test_batched_host_float32():
    from paper_2312_14874_b200 import device as dev
    x = _rows(100, 30000, np.float32, 5)
    out = np.empty_like(x)
    dev.scan_batched_host(x, out)
    want = np.cumsum(x.astype(np.float64), axis=1)
    rel = np.abs(out - want) / np.maximum(np.abs(want), 1e-30)
    assert rel.max() <= 1e-5


def test_batched_host_validation():
    from paper_2312_14874_b200 import device as dev
    with pytest.raises(ValueError):
        dev.scan_batched_host(np.zeros(10, np.int32))
    with pytest.raises(ValueError):
        dev.scan_batched_host(np.zeros((4, 4), np.int32), np.zeros((4, 5), np.int64))
    with pytest.raises(ValueError):
        dev.scan_batched_host(np.zeros((4, 4), np.int64), np.zeros((4, 4), np.int32))
    dev.scan_batched_host(np.zeros((0, 4), np.int32), np.zeros((0, 4), np.int64))


def test_host_workspace_layout_changes_stay_correct():
    """Alternate 1-D and batched host scans with different slot layouts on the
    same device workspace: descriptors must never alias stale slot data."""
    from paper_2312_14874_b200 import core, device as dev
    r = np.random.default_rng(11)
    for it in range(6):
        a = r.integers(0, 5, 3_000_001, dtype=np.int64)
        b = a.copy()
        core.scan_into(b, None, core.full_span(b), 0)
        assert np.array_equal(b, np.cumsum(a)), it
        f = r.random(2_500_003, dtype=np.float32)
        g = np.empty(f.shape, np.float64)
        dev.scan_host(f, g)
        assert np.allclose(g, np.cumsum(f.astype(np.float64)), rtol=1e-12), it
        x = r.integers(0, 9, (700, 3001), dtype=np.int32)
        y = np.empty(x.shape, np.int64)
        dev.scan_batched_host(x, y, chunk_rows=37 + it)
        assert np.array_equal(y, np.cumsum(x, axis=1, dtype=np.int64)), it


@pytest.mark.parametrize("n,dt", [(1 << 24, np.int64), ((1 << 24) + 12345, np.float32), (3 << 22, np.int32)])
def test_host_scan_default_chunks_every_kernel(n, dt):
    """Default chunk sizes put 16-32 MiB chunks through whichever 1-D kernel the
    library picks (stream / rounds / tiles): the workspace scratch must fit all."""
    import contextlib
    from paper_2312_14874_b200 import _lib, core
    lib = _lib.load()
    r = np.random.default_rng(n)
    a = r.integers(0, 100, n).astype(dt) if np.dtype(dt).kind != "f" else r.random(n, dtype=dt)
    want = np.cumsum(a.astype(np.float64 if np.dtype(dt).kind == "f" else np.int64))
    for k in (0, 1, 2, 3):
        prev = lib.ps_get_tuning(b"scan_kernel")
        lib.ps_set_tuning(b"scan_kernel", k)
        try:
            b = a.copy()
            core.scan_into(b, None, core.full_span(b), 0)
        finally:
            lib.ps_set_tuning(b"scan_kernel", prev)
        if np.dtype(dt).kind == "f":
            assert np.max(np.abs(b - want) / np.maximum(want, 1e-30)) <= 1e-6, k
        else:
            assert np.array_equal(b, want.astype(dt)), k

"""ScanEngine / DistributedScanEngine on the GPU (single process): the
reference's engine contract -- schemes, stats, delay hooks, error surface --
with the CUDA library as the local ops."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_scan_engine_all_schemes_cuda_and_numpy():
    import paper_2312_14874_b200 as ps
    from paper_2312_14874_b200.engine import ScanEngine
    a = np.random.default_rng(3).integers(0, 1 << 32, 1_000_003, dtype=np.uint32)
    want = np.cumsum(a, dtype=np.uint64).astype(np.uint32)
    for threads in (1, 4):
        eng = ScanEngine(threads)
        for scheme in ps.SchemeId:
            for block_len in (0, 4096):
                x = torch.from_numpy(a.copy()).cuda()
                total = eng.run(ps.ScanRequest(data=x, scheme=scheme, threads=threads, block_len=block_len,
                                               collect_stats=True))
                assert np.array_equal(x.cpu().numpy(), want), (threads, scheme, block_len)
                assert total == int(a.astype(np.uint64).sum())
                st = eng.last_stats
                assert st.kernel_launches == 1 and st.bytes_moved == 2 * a.nbytes
                h = a.copy()
                out = np.empty_like(h)
                eng.run(ps.ScanRequest(data=h, out=out, scheme=scheme, threads=threads, block_len=block_len))
                assert np.array_equal(out, want) and np.array_equal(h, a)


def test_distributed_engine_single_gpu():
    from paper_2312_14874_b200.distributed import DistributedScanEngine
    from paper_2312_14874_b200.engine import ScanRequest
    from paper_2312_14874_b200.plan import SchemeId
    a = np.random.default_rng(4).random(3_000_001, dtype=np.float32)
    want = np.cumsum(a.astype(np.float64))
    eng = DistributedScanEngine()
    seen = []
    for scheme in SchemeId:
        x = torch.from_numpy(a).cuda()
        out = torch.empty_like(x)
        total = eng.run(ScanRequest(data=x, out=out, scheme=scheme, collect_stats=True,
                                    delay_hook=lambda w, k, ph: seen.append(ph)))
        got = out.cpu().numpy()
        assert np.max(np.abs(got - want) / want) <= 1e-6
        assert abs(total - want[-1]) <= 1e-9 * want[-1]
        assert eng.last_stats.iterations == 1
    assert seen == ["pass1", "pass2"] * len(SchemeId)


def test_engine_worker_failure_is_runtime_error():
    import paper_2312_14874_b200 as ps
    x = torch.arange(10, dtype=torch.int64, device="cuda")

    def boom(w, k, ph):
        if ph == "pass2":
            raise OSError("injected")

    with pytest.raises(RuntimeError) as ei:
        ps.execute(ps.ScanRequest(data=x, delay_hook=boom))
    assert isinstance(ei.value.__cause__, OSError)

"""Benchmark harness + CLI drop-ins, modelled on the
reference's pkg/tests/test_bench.py and test_cli.py.

CPU tests cover the harness logic (config validation, seeded inputs, the
numpy verification oracle pinned against the C restatement of the
reference, CSV schema, sweep bookkeeping, CLI usage errors); GPU tests run
cases and the verification matrix through the CUDA path.
"""

import csv
import io
import statistics

import numpy as np
import pytest

from paper_2312_14874_b200 import bench
from paper_2312_14874_b200.bench import (
    ALGORITHMS,
    CSV_COLUMNS,
    GPU_ALGOS,
    BenchError,
    BenchRecord,
    CaseConfig,
    checksum,
    make_input,
    oracle_scan,
    run_case,
    sweep,
    verify_output,
    write_csv,
)
from paper_2312_14874_b200.cli import main

from conftest import reference_scan


def run_cli(capsys, *argv):
    code = main(list(argv))
    captured = capsys.readouterr()
    return code, captured.out, captured.err


# ---------------------------------------------------------------- CPU: harness logic

def test_config_validation():
    with pytest.raises(ValueError):
        CaseConfig(algo="Quantum")
    with pytest.raises(ValueError):
        CaseConfig(reps=0)
    with pytest.raises(ValueError):
        CaseConfig(reps=4)  # records carry the median of at least 5 reps
    with pytest.raises(ValueError):
        CaseConfig(elem_type="f64")
    with pytest.raises(ValueError):
        CaseConfig(device="tpu")
    for algo in ALGORITHMS:
        CaseConfig(algo=algo)


def test_labels_extend_the_reference_set():
    ref = ("Scalar", "SIMD", "SIMD-V1", "SIMD-V2", "SIMD-T", "Scalar1", "Scalar2", "SIMD1", "SIMD2",
           "Scalar1-P", "Scalar2-P", "SIMD1-P", "SIMD2-P")
    assert ALGORITHMS[:len(ref)] == ref
    assert set(GPU_ALGOS) == set(ALGORITHMS[len(ref):])
    assert CSV_COLUMNS[:12] == ("algo", "elem_type", "n", "threads", "block_len", "d0", "d_last",
                                "out_of_place", "reps", "median_ns", "throughput_eps", "checksum")


def test_default_case_elements_scales_with_threads():
    assert bench.default_case_elements(1) == 1 << 24
    assert bench.default_case_elements(4) == 4 << 24
    assert bench.default_case_elements(16) == 8 << 24  # capped at 8 threads


def test_make_input_deterministic():
    assert np.array_equal(make_input("i32", 1000, 9), make_input("i32", 1000, 9))
    assert np.array_equal(make_input("f32", 1000, 9), make_input("f32", 1000, 9))
    assert not np.array_equal(make_input("i32", 1000, 9), make_input("i32", 1000, 10))
    assert make_input("i32", 10, 0).dtype == np.uint32
    assert make_input("f32", 10, 0).dtype == np.float32


def test_make_input_matches_golden_generator():
    from conftest import make_data

    for elem in ("i32", "f32"):
        assert np.array_equal(make_input(elem, 4096, 5), make_data(elem, 4096, 5))


@pytest.mark.parametrize("elem", ["i32", "f32"])
@pytest.mark.parametrize("n", [0, 1, 17, 4096, 100_003])
def test_oracle_scan_matches_c_restatement(oracle_lib, elem, n):
    """The harness's numpy oracle equals the C restatement of the reference's
    _scan_kernel (oracle/scan_oracle.c) bit for bit."""
    data = make_input(elem, n, 33)
    want = data.copy()
    if n:
        oracle_lib.scan(want, 0, n)
    assert np.array_equal(oracle_scan(data), want)
    assert np.array_equal(oracle_scan(data), reference_scan(data))


def test_verify_output_rejects_corruption():
    data = make_input("i32", 1000, 1)
    good = oracle_scan(data)
    verify_output(good, good, "i32")
    bad = good.copy()
    bad[500] += 1
    with pytest.raises(BenchError, match="index 500"):
        verify_output(bad, good, "i32")
    fgood = oracle_scan(make_input("f32", 1000, 1))
    verify_output(fgood, fgood, "f32")
    fbad = fgood * np.float32(1.001)
    with pytest.raises(BenchError):
        verify_output(fbad, fgood, "f32")
    verify_output(np.empty(0, np.float32), np.empty(0, np.float32), "f32")


def test_checksum_is_crc32_of_bytes():
    import zlib

    a = np.arange(100, dtype=np.uint32)
    assert checksum(a) == zlib.crc32(a.tobytes())
    assert checksum(a[::2]) == zlib.crc32(np.ascontiguousarray(a[::2]).tobytes())


def test_resolved_block_len():
    assert bench._resolved_block_len(CaseConfig(algo="Scalar", block_len=512)) == 0
    assert bench._resolved_block_len(CaseConfig(algo="GPU", block_len=512)) == 0
    assert bench._resolved_block_len(CaseConfig(algo="SIMD1", block_len=512)) == 0
    assert bench._resolved_block_len(CaseConfig(algo="SIMD1-P", block_len=512)) == 512
    assert bench._resolved_block_len(CaseConfig(algo="SIMD1-P")) > 0
    assert bench._resolved_block_len(CaseConfig(algo="SIMD-V1", block_len=0)) == 0


def _record(**kw):
    base = dict(algo="Scalar", elem_type="i32", n=4096, threads=1, block_len=0, d0=1.0, d_last=1.0,
                out_of_place=False, reps=5, rep_times_ns=[5, 4, 3, 2, 1], median_ns=3,
                throughput_eps=1.5e9, checksum=1234, device="cuda", bandwidth_gbs=12.5)
    base.update(kw)
    return BenchRecord(**base)


def test_csv_schema_and_parse():
    recs = [_record(), _record(algo="SIMD1-P", threads=2, block_len=512, out_of_place=True)]
    buf = io.StringIO()
    write_csv(recs, buf)
    text = buf.getvalue()
    assert "\r" not in text and text.endswith("\n")
    rows = list(csv.DictReader(io.StringIO(text)))
    assert list(rows[0].keys()) == list(CSV_COLUMNS)
    assert len(rows) == 2
    assert rows[1]["algo"] == "SIMD1-P"
    assert rows[1]["out_of_place"] == "1"
    assert rows[1]["block_len"] == "512"
    assert rows[0]["device"] == "cuda"
    assert float(rows[0]["bandwidth_gbs"]) == 12.5
    assert int(rows[0]["median_ns"]) == 3


def test_sweep_bookkeeping(monkeypatch):
    seen = []

    def fake(cfg):
        seen.append(cfg)
        if cfg.threads == 3:
            raise BenchError("injected")
        return _record(threads=cfg.threads, d0=cfg.d0, block_len=cfg.block_len)

    monkeypatch.setattr(bench, "run_case", fake)
    records, failures = sweep("threads", [1, 3, 2], CaseConfig(algo="Scalar1", n=4096, reps=5, seed=4))
    assert [r.threads for r in records] == [1, 2]
    assert len(failures) == 1 and failures[0][0] == 3
    assert {c.seed for c in seen} == {4}  # shared seed: every point scans the same data
    records, _ = sweep("dilation", [0.0, 0.5], CaseConfig(algo="Scalar1", n=4096, reps=5))
    assert [r.d0 for r in records] == [0.0, 0.5]
    records, _ = sweep("block_len", [512, 1024], CaseConfig(algo="SIMD1-P", n=4096, reps=5))
    assert [r.block_len for r in records] == [512, 1024]


def test_sweep_validation():
    with pytest.raises(ValueError):
        sweep("voltage", [1], CaseConfig())
    with pytest.raises(ValueError):
        sweep("threads", [], CaseConfig())


def test_cli_unknown_algorithm_is_usage_error(capsys):
    code, _, err = run_cli(capsys, "scan", "--algo", "Warp9")
    assert code == 2
    assert "unknown algorithm" in err


def test_cli_unknown_flag_is_usage_error():
    with pytest.raises(SystemExit) as exc:
        main(["scan", "--frobnicate"])
    assert exc.value.code == 2


def test_cli_bad_reps_is_usage_error(capsys):
    code, _, err = run_cli(capsys, "bench", "--reps", "3", "--n", "16")
    assert code == 2
    assert "reps" in err


def test_cli_sweep_requires_dimension():
    with pytest.raises(SystemExit) as exc:
        main(["sweep", "--grid", "1,2"])
    assert exc.value.code == 2


# ---------------------------------------------------------------- GPU: cases through CUDA

@pytest.mark.gpu
def test_run_case_smoke():
    rec = run_case(CaseConfig(algo="Scalar", elem_type="i32", n=10**5, reps=5, seed=3))
    assert rec.throughput_eps > 0
    assert rec.median_ns > 0
    assert len(rec.rep_times_ns) == 5
    assert rec.median_ns == int(statistics.median(rec.rep_times_ns))
    assert rec.checksum == checksum(oracle_scan(make_input("i32", 10**5, 3)))


@pytest.mark.gpu
@pytest.mark.parametrize("device", ["host", "cuda"])
def test_every_algorithm_checksum_matches_oracle(device):
    n, seed = 30000, 11
    expected_crc = checksum(oracle_scan(make_input("i32", n, seed)))
    for algo in ALGORITHMS:
        threads = 2 if algo in bench.MULTI_THREAD_ALGOS else 1
        rec = run_case(CaseConfig(algo=algo, elem_type="i32", n=n, threads=threads,
                                  block_len=2048, seed=seed, reps=5, device=device))
        assert rec.checksum == expected_crc, algo
        assert rec.device == device


@pytest.mark.gpu
@pytest.mark.parametrize("algo", GPU_ALGOS)
@pytest.mark.parametrize("elem", ["i32", "f32"])
def test_gpu_labels_large_device_resident(algo, elem):
    # above the 32 MiB threshold of the large-input kernels
    rec = run_case(CaseConfig(algo=algo, elem_type=elem, n=(1 << 23) + 5, reps=5, seed=2,
                              device="cuda", out_of_place=True))  # raises unless within FLOAT_RTOL
    if elem == "i32":
        assert rec.checksum == checksum(oracle_scan(make_input(elem, (1 << 23) + 5, 2)))
    # float32: the stream kernel's float-pair path reassociates (<= 1e-6 relative), so the
    # CRC of the result need not equal the sequential oracle's -- as for the reference's
    # own multithreaded float algorithms; run_case has verified the values
    assert rec.bandwidth_gbs > 0


@pytest.mark.gpu
def test_kernel_choice_restored():
    from paper_2312_14874_b200 import _lib

    lib = _lib.load()
    before = lib.ps_get_tuning(b"scan_kernel")
    run_case(CaseConfig(algo="GPU-LB", n=4096, reps=5))
    assert lib.ps_get_tuning(b"scan_kernel") == before


@pytest.mark.gpu
def test_records_deterministic_except_timing():
    cfg = CaseConfig(algo="SIMD", elem_type="f32", n=2**15, seed=21, reps=5)
    a, b = run_case(cfg), run_case(cfg)
    for key in ("algo", "elem_type", "n", "threads", "block_len", "d0", "d_last",
                "out_of_place", "reps", "checksum"):
        assert getattr(a, key) == getattr(b, key)


@pytest.mark.gpu
def test_empty_input_record():
    rec = run_case(CaseConfig(algo="Scalar", n=0, reps=5))
    assert rec.throughput_eps == 0.0
    assert rec.n == 0


@pytest.mark.gpu
def test_cli_scan_total_matches_oracle(capsys):
    code, out, _ = run_cli(capsys, "scan", "--algo", "SIMD1-P", "--n", "16",
                           "--threads", "2", "--elem", "i32", "--seed", "7")
    assert code == 0
    total = int(out.split("total=")[1].split()[0])
    data = make_input("i32", 16, 7)
    assert total == int(data.astype(np.uint64).sum()) & 0xFFFFFFFF
    assert "checksum=" in out


@pytest.mark.gpu
def test_cli_scan_deterministic_output(capsys):
    args = ("scan", "--algo", "GPU", "--n", "1000", "--seed", "3")
    _, first, _ = run_cli(capsys, *args)
    _, second, _ = run_cli(capsys, *args)
    assert first == second


@pytest.mark.gpu
def test_cli_verify_matrix_passes(capsys):
    code, out, _ = run_cli(capsys, "verify", "--n", "4096", "--threads", "2", "--block-len", "512")
    assert code == 0
    assert "all combinations passed" in out
    assert "FAIL" not in out
    assert out.count("PASS") == 2 * 2 * len(ALGORITHMS)


@pytest.mark.gpu
def test_cli_bench_emits_csv(capsys, tmp_path):
    path = tmp_path / "out.csv"
    code, _, _ = run_cli(capsys, "bench", "--algo", "GPU", "--n", "8192", "--device", "cuda",
                         "--csv", str(path))
    assert code == 0
    rows = list(csv.DictReader(path.open()))
    assert len(rows) == 1 and rows[0]["algo"] == "GPU" and rows[0]["device"] == "cuda"


@pytest.mark.gpu
def test_cli_bench_empty_input_notice(capsys):
    code, out, err = run_cli(capsys, "bench", "--algo", "Scalar", "--n", "0")
    assert code == 0
    assert "throughput reported as 0" in err
    rows = list(csv.DictReader(io.StringIO(out)))
    assert rows[0]["throughput_eps"] == "0.0"


@pytest.mark.gpu
def test_cli_sweep_csv(capsys):
    code, out, _ = run_cli(capsys, "sweep", "--dimension", "dilation", "--grid", "0,0.5,1.0",
                           "--algo", "Scalar1", "--n", "8192", "--threads", "2")
    assert code == 0
    rows = list(csv.DictReader(io.StringIO(out)))
    assert [r["d0"] for r in rows] == ["0.0", "0.5", "1.0"]

"""Pin the C oracle (oracle/scan_oracle.c) to the reference's own outputs.

Every golden case (tests/golden/, produced by running the unmodified
reference) is replayed through the oracle; arrays and returned totals must
match bit for bit, float totals included.  This is what lets the GPU parity
tests trust the oracle at sizes where the golden file holds no vector.
"""

import numpy as np
import pytest

from golden_cases import case_id, cases, total_of

ALL = list(cases())


def _same_total(got, want, dtype):
    if want is None:
        return True
    if isinstance(want, float):
        return float(got) == want or (np.isnan(want) and np.isnan(float(got)))
    return int(got) == want


@pytest.mark.parametrize("case", [c for c, _, _ in ALL], ids=[case_id(c) for c, _, _ in ALL])
def test_oracle_matches_reference_golden(case, oracle_lib):
    o = oracle_lib
    _, arrays = __import__("golden_cases").load()
    inp, want = arrays[case["in"]], arrays[case["out"]]
    op = case["op"]
    work = inp.copy()
    total = None
    if op == "sequential_inclusive_scan":
        total = o.scan(work, case["start"], case["len"], case["offset"])
    elif op == "sequential_accumulate":
        total = o.accumulate(work, case["start"], case["len"])
    elif op == "sequential_increment":
        o.increment(work, case["start"], case["len"], case["offset"])
    elif op == "exclusive_from_inclusive":
        total = o.exclusive_from_inclusive(work, case["identity"])
    elif op == "horizontal_scan":
        if case["out_of_place"]:
            out = np.zeros_like(inp)
            total = o.horizontal(work, case["start"], case["len"], case["offset"], case["w"], out=out)
            assert np.array_equal(work, inp)
            work = out
        else:
            total = o.horizontal(work, case["start"], case["len"], case["offset"], case["w"])
    elif op == "vertical_scan":
        total = o.vertical_scan(work, case["start"], case["len"], case["offset"], case["w"],
                                case["scan_in_pass1"], case["block_len"])
    elif op == "tree_scan":
        total = o.tree_scan(work, case["start"], case["len"], case["offset"])
    elif op == "tree_scan_auto":
        total = o.tree_scan_auto(work, case["start"], case["len"], case["offset"], case["w"],
                                 case["block_len"])
    elif op == "engine":
        out = np.empty_like(inp)
        total = o.engine_scan(work, out, threads=case["threads"], scheme=case["scheme"],
                              block_len=case["block_len"])
        work = out
    elif op == "widen_exclusive":
        work, total = o.scan_widen_i32_i64(inp, exclusive=True)
    elif op == "rows_widen_inclusive":
        work = o.rows_scan_widen_i32_i64(inp, threads=3, simd_w=16)
    else:
        pytest.fail(f"unknown golden op {op}")
    assert work.dtype == want.dtype and work.shape == want.shape
    assert np.array_equal(work.view(np.uint8), want.view(np.uint8)), f"array mismatch {case_id(case)}"
    assert _same_total(total, total_of(case), inp.dtype), (total, total_of(case))


def test_golden_covers_every_hot_path_op():
    ops = {c["op"] for c, _, _ in ALL}
    assert {"sequential_inclusive_scan", "sequential_accumulate", "sequential_increment",
            "exclusive_from_inclusive", "horizontal_scan", "vertical_scan", "tree_scan",
            "tree_scan_auto", "engine", "widen_exclusive", "rows_widen_inclusive"} <= ops
    dtypes = {c["dtype"] for c, _, _ in ALL}
    assert {"uint32", "float32", "int64", "int32"} <= dtypes


def test_oracle_engine_many_threads_matches_sequential(oracle_lib):
    """The CPU-baseline port at host-scale thread counts equals the sequential oracle."""
    rng = np.random.default_rng(5)
    for dt, gen in ((np.int64, lambda n: rng.integers(0, 1001, n, dtype=np.int64)),
                    (np.float32, lambda n: rng.random(n, dtype=np.float32))):
        data = gen(1_000_003)
        want = data.copy()
        wt = oracle_lib.scan(want, 0, want.shape[0], 0)
        for scheme in ("accumulate-scan+1", "scan-increment+1", "accumulate-scan", "scan-increment"):
            for threads, block in ((7, 0), (16, 4096), (64, 1 << 14)):
                out = np.empty_like(data)
                t = oracle_lib.engine_scan(data, out, threads=threads, scheme=scheme, block_len=block)
                if dt == np.int64:
                    assert np.array_equal(out, want), (scheme, threads, block)
                    assert t == wt
                else:
                    e = want.astype(np.float64)
                    assert np.max(np.abs(out - e) / np.maximum(e, 1e-30)) <= 1e-5

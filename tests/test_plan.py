"""The planner restatement (paper_2312_14874_b200.plan) against the reference
planner's own output (tests/golden/make_plan.py: compute_grid for 6336
parameter combinations, compute_layout incl. start offsets and
need_last_total, default_block_len), plus the reference's planner tests'
invariants (pkg/tests/test_plan.py) restated."""

import gzip
import json
import os

import pytest

from paper_2312_14874_b200.plan import (CacheInfo, Dilation, SchemeId, compute_grid, compute_layout,
                                        default_block_len, equal_shards)

HERE = os.path.dirname(os.path.abspath(__file__))
with gzip.open(os.path.join(HERE, "golden", "plan_golden.json.gz"), "rt") as f:
    GOLD = json.load(f)


def lay(l):
    return {"spans": [[s.start, s.len] for s in l.spans],
            "pass1": [[it.thread, it.span_index, it.role.value, bool(it.seeded)] for it in l.pass1],
            "pass2": [[it.thread, it.span_index, it.role.value, bool(it.seeded)] for it in l.pass2],
            "scheme": l.scheme.value, "threads": l.threads}


def test_grids_match_reference():
    bad = []
    for case in GOLD["grids"]:
        n, m, scheme, dil, bl, w = case["args"]
        g = compute_grid(n, m, SchemeId(scheme), Dilation(*dil), bl, w)
        got = {"regions": [[r.start, r.len] for r in g.regions], "iterations": g.iterations,
               "layouts": [lay(l) for l in g.layouts]}
        want = {k: case[k] for k in ("regions", "iterations", "layouts")}
        if got != want:
            bad.append(case["args"])
    assert not bad, f"{len(bad)} grids differ, e.g. {bad[:3]}"
    assert len(GOLD["grids"]) > 6000


def test_layouts_match_reference():
    for case in GOLD["layouts"]:
        n, m, scheme, dil, w, start, need = case["args"]
        l = compute_layout(n, m, SchemeId(scheme), Dilation(*dil), w, start=start, need_last_total=need)
        assert lay(l) == case["layout"], case["args"]


def test_default_block_len_matches_reference():
    for case in GOLD["block_len"]:
        l2, tpc, w, explicit = case["args"]
        assert default_block_len(CacheInfo(l2_bytes=l2, threads_per_core=tpc), explicit, w) == case["block_len"], \
            case["args"]


def test_dilation_validation():
    for bad in (-0.1, 1.5):
        with pytest.raises(ValueError):
            Dilation(d0=bad)
        with pytest.raises(ValueError):
            Dilation(d_last=bad)
    with pytest.raises(ValueError):
        compute_layout(-1, 2, SchemeId.SCAN_INCREMENT_EQUAL)
    with pytest.raises(ValueError):
        compute_grid(10, 2, SchemeId.SCAN_INCREMENT_EQUAL, block_len=-1)


@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 10**6 + 7])
@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_equal_shards_exact_cover(n, parts):
    sh = equal_shards(n, parts, align=4)
    assert len(sh) == parts and sum(s.len for s in sh) == n
    pos = 0
    for s in sh:
        assert s.start == pos
        pos += s.len

"""Golden layouts/grids from the UNMODIFIED reference planner (plan.py:131-241,
331-346), so tests/test_plan.py pins paper_2312_14874_b200.plan without the
reference present:

    NUMBA_CACHE_DIR=/tmp/numba_ref PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_plan.py
"""

from __future__ import annotations

import gzip
import itertools
import json
import os

from prefixscan.plan import CacheInfo, Dilation, SchemeId, compute_grid, compute_layout, default_block_len

HERE = os.path.dirname(os.path.abspath(__file__))


def lay(l):
    return {"spans": [[s.start, s.len] for s in l.spans],
            "pass1": [[it.thread, it.span_index, it.role.value, bool(it.seeded)] for it in l.pass1],
            "pass2": [[it.thread, it.span_index, it.role.value, bool(it.seeded)] for it in l.pass2],
            "scheme": l.scheme.value, "threads": l.threads}


def main():
    grids, layouts, blocks = [], [], []
    for n, m, scheme, dil, w, bl in itertools.product(
            (0, 1, 7, 100, 1000, 4096, 100003), (1, 2, 3, 4, 8), list(SchemeId),
            ((1.0, 1.0), (0.5, 1.0), (0.0, 1.0), (0.3, 0.7)), (1, 4, 16), (0, 64, 1000, 12500)):
        if bl and n // (bl * m) > 40:
            continue  # keep the fixture small: at most ~40 iterations per grid
        g = compute_grid(n, m, scheme, Dilation(*dil), bl, w)
        grids.append({"args": [n, m, scheme.value, list(dil), bl, w],
                      "regions": [[r.start, r.len] for r in g.regions], "iterations": g.iterations,
                      "layouts": [lay(l) for l in g.layouts]})
    for n, m, scheme, w, start, need in itertools.product((5, 64, 999, 65537), (1, 2, 5), list(SchemeId), (1, 8),
                                                         (0, 13), (False, True)):
        l = compute_layout(n, m, scheme, Dilation(0.75, 0.25), w, start=start, need_last_total=need)
        layouts.append({"args": [n, m, scheme.value, [0.75, 0.25], w, start, need], "layout": lay(l)})
    for l2, tpc, w, explicit in itertools.product((None, 1 << 20, 2 << 20, 3 << 19), (1, 2), (1, 4, 16), (None, 1, 4)):
        info = CacheInfo(l2_bytes=l2, threads_per_core=tpc)
        blocks.append({"args": [l2, tpc, w, explicit], "block_len": default_block_len(info, explicit, w)})
    with gzip.open(os.path.join(HERE, "plan_golden.json.gz"), "wt") as f:
        json.dump({"grids": grids, "layouts": layouts, "block_len": blocks}, f, separators=(",", ":"))
    print(len(grids), len(layouts), len(blocks))


if __name__ == "__main__":
    main()

"""Loader for the committed golden vectors (tests/golden/, made by make_golden.py
from the unmodified reference).  Shared by the oracle pin and the GPU parity
tests."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=1)
def load():
    with open(os.path.join(GOLDEN_DIR, "manifest.json")) as fh:
        manifest = json.load(fh)
    arrays = dict(np.load(os.path.join(GOLDEN_DIR, "golden.npz")))
    return manifest["cases"], arrays


def cases(op=None):
    all_cases, arrays = load()
    for c in all_cases:
        if op is None or c["op"] == op:
            yield c, arrays[c["in"]], arrays[c["out"]]


def total_of(case):
    t = case.get("total")
    if t is None:
        return None
    if t["kind"] == "float":
        return float.fromhex(t["hex"])
    return int(t["dec"])


def case_id(c):
    keys = ("op", "dtype", "n", "start", "len", "offset", "w", "scheme", "threads", "block_len",
            "scan_in_pass1", "out_of_place")
    return "-".join(f"{c[k]}" for k in keys if k in c) + f"#{c['id']}"

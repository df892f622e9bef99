"""Known-answer tests of the lane primitives (simd.py host models of the warp
scan), after the reference's pkg/tests/test_simd.py:31-61: the zero-filling
lane shift, the Hillis-Steele vector scan taking exactly log2(w) rounds, its
agreement with the sequential scan, and power-of-two validation.  CPU only:
these are the host models; the same rounds run as __shfl_up_sync in every
kernel (checked on the GPU by the parity suite)."""

import numpy as np
import pytest

from conftest import make_data
from paper_2312_14874_b200.simd import (
    SUPPORTED_LANE_WIDTHS,
    AddRoundCounter,
    lane_shift_with_zero_fill,
    vector_inclusive_scan,
)


def test_shift_by_one_zero_fills_lane_zero():
    v = np.array([1, 2, 3, 4], dtype=np.uint32)
    assert lane_shift_with_zero_fill(v, 1).tolist() == [0, 1, 2, 3]


def test_shift_by_zero_is_identity_and_full_width_is_all_zero():
    v = np.array([9, 8, 7, 6], dtype=np.uint32)
    assert lane_shift_with_zero_fill(v, 0).tolist() == [9, 8, 7, 6]
    assert lane_shift_with_zero_fill(v, 4).tolist() == [0, 0, 0, 0]


@pytest.mark.parametrize("k", [-1, 5, 17])
def test_shift_outside_the_vector_is_rejected(k):
    with pytest.raises(ValueError):
        lane_shift_with_zero_fill(np.arange(4, dtype=np.uint32), k)


def test_shift_keeps_dtype_and_leaves_input_alone():
    v = np.array([1.5, 2.5, 3.5, 4.5], dtype=np.float32)
    out = lane_shift_with_zero_fill(v, 2)
    assert out.dtype == np.float32 and out.tolist() == [0.0, 0.0, 1.5, 2.5]
    assert v.tolist() == [1.5, 2.5, 3.5, 4.5]


@pytest.mark.parametrize("w", SUPPORTED_LANE_WIDTHS)
def test_vector_scan_takes_log2_w_rounds(w):
    counter = AddRoundCounter()
    out = vector_inclusive_scan(np.ones(w, dtype=np.uint32), counter)
    assert counter.rounds == w.bit_length() - 1
    assert out.tolist() == list(range(1, w + 1))


@pytest.mark.parametrize("w", SUPPORTED_LANE_WIDTHS)
def test_vector_scan_equals_the_sequential_scan(w, oracle_lib):
    v = make_data("i32", w, seed=w)
    want = v.copy()
    oracle_lib.scan(want, 0, w, 0)  # the reference's _scan_kernel, restated (core.py:86-92)
    assert np.array_equal(vector_inclusive_scan(v), want)


@pytest.mark.parametrize("w", SUPPORTED_LANE_WIDTHS)
def test_vector_scan_wraps_uint32_like_the_element_dtype(w):
    v = np.full(w, 0xFFFFFFFF, dtype=np.uint32)
    got = vector_inclusive_scan(v)
    want = (np.arange(1, w + 1, dtype=np.uint64) * 0xFFFFFFFF) & 0xFFFFFFFF
    assert got.dtype == np.uint32 and got.tolist() == want.astype(np.uint32).tolist()


@pytest.mark.parametrize("n", [3, 6, 12])
def test_vector_scan_rejects_non_power_of_two(n):
    with pytest.raises(ValueError):
        vector_inclusive_scan(np.ones(n, dtype=np.uint32))


def test_counter_accumulates_over_calls():
    counter = AddRoundCounter()
    vector_inclusive_scan(np.ones(8, dtype=np.uint32), counter)
    vector_inclusive_scan(np.ones(16, dtype=np.uint32), counter)
    assert counter.rounds == 3 + 4

"""The P5 certification helper (tests/parity.py) itself: identical sets pass, a near-tie swap
within 2 max|dx| is certified, anything else fails (CPU)."""
import numpy as np
import pytest

from parity import certify_sets, walk_chain


def test_identical_sets():
    x = np.array([3.0, -2.0, 1.0, 0.5])
    assert certify_sets([0, 1], [0, 1], x, x)


def test_certified_near_tie():
    x_ref = np.array([3.0, 2.0, 1.0 + 1e-7, 1.0])
    x_gpu = x_ref.copy()
    x_gpu[2] = 1.0 - 1e-7                      # the GPU's rounding flips the order of 2 and 3
    assert certify_sets([0, 1, 3], [0, 1, 2], x_gpu, x_ref) is False
    assert walk_chain([("a", [0], [0], x_ref, x_ref), ("b", [0, 1, 3], [0, 1, 2], x_gpu, x_ref),
                       ("c", [9], [0], x_ref, x_ref)]) == "b"     # stops at the first certified swap


def test_uncertified_swap_fails():
    x = np.array([3.0, 2.0, 1.5, 1.0])
    with pytest.raises(AssertionError, match="uncertified"):
        certify_sets([0, 1, 3], [0, 1, 2], x + 1e-9, x)          # 1.5 vs 1.0 is no near-tie
    with pytest.raises(AssertionError, match="kept counts"):
        certify_sets([0, 1], [0, 1, 2], x, x)
    with pytest.raises(AssertionError):
        walk_chain([("h1", [0, 3], [0, 1], x, x)])

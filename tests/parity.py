"""Shared parity helpers for the GPU tests (no method arithmetic of its own beyond comparisons).

P5 certification (parity protocol row P5): when the oracle runs a chain from
the same inputs, its kept index sets must equal the GPU's at every site, except for swaps
between near-tied magnitudes.  A swap of i (in one set) against j (in the other) is certified
only if  ||x_i| - |x_j||  (oracle values)  <=  2 * max_m |x_gpu_m - x_oracle_m|  of THAT site's
vector.  Anything else is a selection bug and fails the test.  After the first certified swap
the two chains legitimately diverge, so the caller stops comparing downstream sites and
reports the swap (a skip whose reason names the site and the margin).
"""
import numpy as np


def certify_sets(idx_gpu, idx_ref, x_gpu, x_ref, where=""):
    """True if the index sets are identical; False if they differ only by certified near-tie
    swaps; AssertionError otherwise (P5)."""
    a = np.asarray(idx_gpu, dtype=np.int64)
    b = np.asarray(idx_ref, dtype=np.int64)
    if a.shape == b.shape and np.array_equal(a, b):
        return True
    assert a.shape == b.shape, f"{where}: kept counts differ ({a.size} vs {b.size})"
    x_gpu = np.asarray(x_gpu, dtype=np.float64)
    x_ref = np.asarray(x_ref, dtype=np.float64)
    tol = 2.0 * float(np.max(np.abs(x_gpu - x_ref)))
    only_gpu = np.setdiff1d(a, b)
    only_ref = np.setdiff1d(b, a)
    assert only_gpu.size == only_ref.size and only_gpu.size > 0, f"{where}: malformed index lists"
    mg = np.abs(x_ref[only_gpu])[:, None]
    mr = np.abs(x_ref[only_ref])[None, :]
    gap = float(np.max(np.abs(mg - mr)))
    assert gap <= tol, (f"{where}: uncertified Top-K difference: {only_gpu.size} swap(s), "
                        f"max ||x_i|-|x_j|| = {gap:.3e} > 2 max|dx| = {tol:.3e} (P5)")
    return False


def walk_chain(sites):
    """``sites``: iterable of (name, idx_gpu, idx_ref, x_gpu, x_ref) in execution order.
    Returns None if every site's index set agrees, else the name of the first site with a
    certified near-tie swap (uncertified differences raise)."""
    for name, ig, ir, xg, xr in sites:
        if not certify_sets(ig, ir, xg, xr, where=name):
            return name
    return None

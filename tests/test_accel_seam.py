"""Seam A: ``paper_1802_03749_b200.accel`` as a ``meshplan._accel`` backend.

Runs the reference's OWN backend-equivalence tests
(/root/reference/pkg/tests/test_accel_backends.py:41-100) with this package's
backend in the place of ``numba_impl``: every one of the eight callables must
equal the reference ``numpy_impl`` bit for bit (pair order excepted, as the
reference allows).  Then the same comparison on larger random inputs.
Host-side C ABI only (no GPU); skipped where /root/reference is absent (the
GPU box), since the reference itself is the checker.
"""

import importlib.util
import os
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1802_03749_b200 import accel

REF = Path("/root/reference/pkg")
pytestmark = pytest.mark.skipif(not (REF / "tests" / "test_accel_backends.py").exists(),
                                reason="the reference package is the checker (build container only)")


@pytest.fixture(scope="module")
def ref_tests():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_meshplan")
    sys.dont_write_bytecode = True
    if str(REF / "src") not in sys.path:
        sys.path.insert(0, str(REF / "src"))
    spec = importlib.util.spec_from_file_location("ref_test_accel_backends", REF / "tests" / "test_accel_backends.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.numba_impl = accel  # the reference's "second backend" is this one
    return mod


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("least_loaded", [True, False])
def test_reference_greedy_colour_csr_equal(ref_tests, seed, least_loaded):
    ref_tests.test_greedy_colour_csr_equal(seed, least_loaded)


@pytest.mark.parametrize("seed", [3, 4])
def test_reference_greedy_colour_adj_and_order_equal(ref_tests, seed):
    ref_tests.test_greedy_colour_adj_and_order_equal(seed)


@pytest.mark.parametrize("seed", [5, 6])
def test_reference_bfs_equal(ref_tests, seed):
    ref_tests.test_bfs_equal(seed)


@pytest.mark.parametrize("seed", [7, 8])
def test_reference_matching_and_refine_equal(ref_tests, seed):
    ref_tests.test_matching_and_refine_equal(seed)


def test_reference_pairs_from_segments_equal_as_sets(ref_tests):
    ref_tests.test_pairs_from_segments_equal_as_sets()


# ---- larger inputs, every callable vs numpy_impl ------------------------------------------


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_every_callable_matches_numpy_impl_on_larger_graphs(ref_tests, seed):
    ref = ref_tests.numpy_impl
    n = 2000
    indptr, indices, weights = ref_tests.random_graph(n, seed)
    # colouring
    cp, ci = ref_tests.random_csr(3000, 700, seed, per_row=4)
    for ll in (True, False):
        assert np.array_equal(accel.greedy_colour_csr(cp, ci, 700, ll), ref.greedy_colour_csr(cp, ci, 700, ll))
    order = ref.smallest_last_order(indptr, indices)
    assert np.array_equal(accel.smallest_last_order(indptr, indices), order)
    for ll in (True, False):
        assert np.array_equal(accel.greedy_colour_adj(indptr, indices, order, ll),
                              ref.greedy_colour_adj(indptr, indices, order, ll))
    # BFS (levels, traversal order, count), from several starts
    for start in (0, n // 2, n - 1):
        la, qa, ta = accel.bfs_levels(indptr, indices, start)
        lb, qb, tb = ref.bfs_levels(indptr, indices, start)
        assert ta == tb and np.array_equal(la, lb) and np.array_equal(qa[:ta], qb[:tb])
    # matching, refinement (in place), cut
    node_w = np.random.default_rng(seed).integers(1, 4, n).astype(np.int64)
    visit = np.random.default_rng(seed + 1).permutation(n).astype(np.int64)
    assert np.array_equal(accel.heavy_edge_matching(indptr, indices, weights, node_w, visit, 6),
                          ref.heavy_edge_matching(indptr, indices, weights, node_w, visit, 6))
    k = 16
    a0 = (np.arange(n) * k // n).astype(np.int64)
    for use_w in (True, False):
        a, b = a0.copy(), a0.copy()
        bw_a = np.bincount(a, weights=node_w, minlength=k).astype(np.int64)
        bw_b = bw_a.copy()
        cap = int(bw_a.max()) + 3
        for _ in range(3):
            ma = accel.refine_boundary_pass(indptr, indices, weights, a, bw_a, node_w, cap, use_w)
            mb = ref.refine_boundary_pass(indptr, indices, weights, b, bw_b, node_w, cap, use_w)
            assert ma == mb
            assert np.array_equal(a, b) and np.array_equal(bw_a, bw_b)
            assert accel.cut_weight(indptr, indices, weights, a, use_w) == ref.cut_weight(indptr, indices, weights,
                                                                                         b, use_w)
    # pairs (multiset)
    sp, sv = ref_tests.random_csr(400, 300, seed, per_row=7)
    ua, va = accel.pairs_from_segments(sp, sv)
    ub, vb = ref.pairs_from_segments(sp, sv)
    assert (ua < va).all()
    assert sorted(zip(ua.tolist(), va.tolist())) == sorted(zip(ub.tolist(), vb.tolist()))


def test_edge_cases(ref_tests):
    ref = ref_tests.numpy_impl
    # empty segments / single-member segments give no pairs
    us, vs = accel.pairs_from_segments(np.array([0, 0, 1, 1]), np.array([5]))
    assert us.size == 0 and vs.size == 0
    # isolated start node
    ip = np.array([0, 0, 1, 2], dtype=np.int64)
    ix = np.array([2, 1], dtype=np.int64)
    la, qa, ta = accel.bfs_levels(ip, ix, 0)
    lb, qb, tb = ref.bfs_levels(ip, ix, 0)
    assert ta == tb == 1 and np.array_equal(la, lb)
    # refine_boundary_pass needs writeable int64 arrays (it mutates them), like the reference
    with pytest.raises(TypeError):
        accel.refine_boundary_pass(ip, ix, np.ones(2, dtype=np.int64), np.zeros(3, dtype=np.int32),
                                   np.zeros(1, dtype=np.int64), np.ones(3, dtype=np.int64), 5, True)

"""Native (host C++) k-way partitioner kernels vs the oracle restatement.

These run on the CPU: the sequential sweeps of the reference partitioner
are host code in the native library (no GPU needed)."""

import numpy as np
import pytest

from paper_1802_03749_b200 import _native
from oracle import kway


def _graph(seed, n=None):
    rng = np.random.default_rng(seed)
    n = n or int(rng.integers(8, 160))
    dense = np.triu(rng.random((n, n)) < rng.uniform(0.02, 0.2), 1)
    w = np.triu(rng.integers(1, 4, (n, n)), 1) * dense
    w = w + w.T
    indptr = np.concatenate(([0], np.cumsum((w > 0).sum(1)))).astype(np.int64)
    rows, cols = np.nonzero(w)
    return indptr, cols.astype(np.int64), w[rows, cols].astype(np.int64), rng


def p(a):
    return a.ctypes.data


@pytest.mark.parametrize("seed", range(10))
def test_heavy_edge_matching(seed):
    ip, ix, w, rng = _graph(seed)
    n = len(ip) - 1
    nw = rng.integers(1, 4, n).astype(np.int64)
    visit = rng.permutation(n).astype(np.int64)
    out = np.empty(n, dtype=np.int64)
    _native.call("mp_heavy_edge_matching", n, p(ip), p(ix), p(w), p(nw), p(visit), 4, p(out))
    assert np.array_equal(out, kway.heavy_edge_matching(ip, ix, w, nw, visit, 4))


@pytest.mark.parametrize("seed", range(10))
def test_initial_partition_rebalance_refine(seed):
    ip, ix, w, rng = _graph(seed)
    n = len(ip) - 1
    nw = rng.integers(1, 3, n).astype(np.int64)
    nb = int(rng.integers(2, 7))
    cap = int(nw.sum() // nb + rng.integers(0, 3))
    a = np.empty(n, dtype=np.int64)
    _native.call("mp_initial_partition", n, p(ip), p(ix), p(nw), nb, cap, p(a))
    want = kway.initial_partition(ip, ix, nw, nb, cap)
    assert np.array_equal(a, want)
    for use_w in (1, 0):
        a1, a2 = a.copy(), a.copy()
        bw1 = np.bincount(a1, weights=nw, minlength=nb).astype(np.int64)
        bw2 = bw1.copy()
        _native.call("mp_rebalance", n, p(ip), p(ix), p(w), p(a1), p(bw1), nb, p(nw), cap, use_w)
        kway.rebalance(ip, ix, w, a2, bw2, nw, cap, use_w)
        assert np.array_equal(a1, a2) and np.array_equal(bw1, bw2)
        moves = np.zeros(1, dtype=np.int64)
        _native.call("mp_refine_boundary_pass", n, p(ip), p(ix), p(w), p(a1), p(bw1), nb, p(nw), cap, use_w,
                     p(moves))
        m2 = kway.refine_boundary_pass(ip, ix, w, a2, bw2, nw, cap, use_w)
        assert int(moves[0]) == m2 and np.array_equal(a1, a2) and np.array_equal(bw1, bw2)
        cut = np.zeros(1, dtype=np.int64)
        _native.call("mp_cut_weight", n, p(ip), p(ix), p(w), p(a1), use_w, p(cut))
        assert int(cut[0]) == kway.cut_weight(ip, ix, w, a1, use_w)


def test_round_half_even_target():
    # total*k1/(k1+k2) = 2.5 -> Python round() gives 2 (half to even)
    ip = np.array([0, 0, 0, 0, 0, 0], dtype=np.int64)
    ix = np.zeros(0, dtype=np.int64)
    nw = np.ones(5, dtype=np.int64)
    a = np.empty(5, dtype=np.int64)
    _native.call("mp_initial_partition", 5, p(ip), p(ix), p(nw), 2, 5, p(a))
    assert np.array_equal(a, kway.initial_partition(ip, ix, nw, 2, 5))
    assert np.bincount(a).tolist() == [2, 3]  # round(2.5) == 2, not 3


@pytest.mark.parametrize("seed", range(40))
def test_rebalance_overloaded_random_assignments(seed):
    """Unbalanced starting assignments (several over-cap blocks, some with no
    room anywhere nearby): native rebalance == the reference restatement."""
    ip, ix, w, rng = _graph(seed, n=int(np.random.default_rng(seed).integers(20, 240)))
    n = len(ip) - 1
    nw = rng.integers(1, 4, n).astype(np.int64)
    nb = int(rng.integers(2, 12))
    skew = rng.dirichlet(np.full(nb, 0.4))
    a = rng.choice(nb, size=n, p=skew).astype(np.int64)
    cap = int(max(1, nw.sum() // nb + rng.integers(-1, 4)))
    for use_w in (1, 0):
        a1, a2 = a.copy(), a.copy()
        bw1 = np.bincount(a1, weights=nw, minlength=nb).astype(np.int64)
        bw2 = bw1.copy()
        _native.call("mp_rebalance", n, p(ip), p(ix), p(w), p(a1), p(bw1), nb, p(nw), cap, use_w)
        kway.rebalance(ip, ix, w, a2, bw2, nw, cap, use_w)
        assert np.array_equal(a1, a2) and np.array_equal(bw1, bw2)


@pytest.mark.parametrize("seed", range(30))
def test_refine_boundary_frontier_equals_repeated_passes(seed):
    """mp_refine_boundary (frontier-only later sweeps) == up to 8 full
    reference sweeps (partition.py:329-338) from skewed random assignments."""
    ip, ix, w, rng = _graph(seed, n=int(np.random.default_rng(seed + 100).integers(20, 300)))
    n = len(ip) - 1
    nw = rng.integers(1, 3, n).astype(np.int64)
    nb = int(rng.integers(2, 10))
    a = rng.choice(nb, size=n, p=rng.dirichlet(np.full(nb, 2.0))).astype(np.int64)
    cap = int(max(1, nw.sum() // nb + rng.integers(0, 6)))
    for use_w in (1, 0):
        a1, a2 = a.copy(), a.copy()
        bw1 = np.bincount(a1, weights=nw, minlength=nb).astype(np.int64)
        bw2 = bw1.copy()
        total = 0
        for _ in range(8):
            m = kway.refine_boundary_pass(ip, ix, w, a2, bw2, nw, cap, use_w)
            total += m
            if m == 0:
                break
        moves = np.zeros(1, dtype=np.int64)
        _native.call("mp_refine_boundary", n, p(ip), p(ix), p(w), p(a1), p(bw1), nb, p(nw), cap, use_w, 8, p(moves))
        assert np.array_equal(a1, a2) and np.array_equal(bw1, bw2) and int(moves[0]) == total


@pytest.mark.parametrize("seed", range(3))
def test_refine_boundary_threaded_first_sweep(seed):
    """Graphs above the threaded pre-scan threshold (2^16 nodes): the same
    result as repeated full single sweeps (each checked against the oracle
    above)."""
    rng = np.random.default_rng(seed)
    side = 300
    n = side * side
    idx = np.arange(n).reshape(side, side)
    pairs = np.concatenate([np.stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()], 1),
                            np.stack([idx[:-1, :].ravel(), idx[1:, :].ravel()], 1)])
    wts = rng.integers(1, 4, len(pairs))
    src = np.concatenate([pairs[:, 0], pairs[:, 1]])
    dst = np.concatenate([pairs[:, 1], pairs[:, 0]])
    ww = np.concatenate([wts, wts])
    order = np.lexsort((dst, src))
    ix, w = dst[order].astype(np.int64), ww[order].astype(np.int64)
    ip = np.concatenate(([0], np.cumsum(np.bincount(src, minlength=n)))).astype(np.int64)
    nw = np.ones(n, dtype=np.int64)
    nb = 300
    a = np.minimum((np.arange(n) + rng.integers(-200, 200, n)) // (n // nb), nb - 1).clip(0).astype(np.int64)
    cap = n // nb + 20
    for use_w in (1, 0):
        a1, a2 = a.copy(), a.copy()
        bw1 = np.bincount(a1, weights=nw, minlength=nb).astype(np.int64)
        bw2 = bw1.copy()
        total, moves = 0, np.zeros(1, dtype=np.int64)
        for _ in range(8):
            _native.call("mp_refine_boundary_pass", n, p(ip), p(ix), p(w), p(a2), p(bw2), nb, p(nw), cap, use_w,
                         p(moves))
            total += int(moves[0])
            if moves[0] == 0:
                break
        assert total > 0
        _native.call("mp_refine_boundary", n, p(ip), p(ix), p(w), p(a1), p(bw1), nb, p(nw), cap, use_w, 8, p(moves))
        assert np.array_equal(a1, a2) and np.array_equal(bw1, bw2) and int(moves[0]) == total

"""Seam A: a drop-in ``meshplan._accel`` backend over the native library.

The reference dispatches its planning kernels through ``meshplan._accel``
(pkg/src/meshplan/_accel/__init__.py:43-50), which exports exactly these
eight callables from ``numba_impl`` or ``numpy_impl``, bit-identical to each
other (numpy_impl.py:1-6; test_accel_backends.py:41-100).  This module is a
third backend with the same signatures, the same dtypes (int64 arrays in,
new int64 arrays out; ``refine_boundary_pass`` mutates ``assignment`` and
``block_weights`` in place) and the same results, calling the C ABI in
``include/meshplan_b200.h``:

=========================  ======================================  ====================
callable                   reference                               C ABI
=========================  ======================================  ====================
greedy_colour_csr          numpy_impl.py:12-60                     mp_greedy_colour_csr
greedy_colour_adj          numpy_impl.py:62-92                     mp_greedy_colour_adj
smallest_last_order        numpy_impl.py:95-111                    mp_smallest_last_order
bfs_levels                 numpy_impl.py:114-131                   mp_bfs_levels_host
heavy_edge_matching        numpy_impl.py:134-157                   mp_heavy_edge_matching
refine_boundary_pass       numpy_impl.py:160-194                   mp_refine_boundary_pass
cut_weight                 numpy_impl.py:197-206                   mp_cut_weight
pairs_from_segments        numpy_impl.py:209-259                   mp_pairs_from_segments
=========================  ======================================  ====================

These are the reference's host-array entry points (sequential by
definition, or per-call small); the plan builder itself uses the device
variants (GPU BFS, matching in dependency rounds, per-block colouring on the
GPU) on device-resident arrays.  INTEGRATION.md shows the two-line dispatch
change that makes ``meshplan._accel`` pick this module.
"""

import numpy as np

from . import _native
from .colouring import greedy_colour_adj, greedy_colour_csr, smallest_last_order

__all__ = ["backend", "greedy_colour_csr", "greedy_colour_adj", "smallest_last_order", "bfs_levels",
           "heavy_edge_matching", "refine_boundary_pass", "cut_weight", "pairs_from_segments"]


def backend() -> str:
    """Name of this backend (``_accel.backend()``, _accel/__init__.py:38-40)."""
    return "b200"


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def bfs_levels(indptr, indices, start):
    """``(levels, visit_order, n_visited)``: FIFO BFS from ``start``, -1 for
    unreached nodes; the first ``n_visited`` entries of ``visit_order`` are
    the traversal order (numpy_impl.py:114-131)."""
    indptr, indices = _i64(indptr), _i64(indices)
    n = len(indptr) - 1
    levels = np.empty(n, dtype=np.int64)
    queue = np.empty(n, dtype=np.int64)
    tail = np.zeros(1, dtype=np.int64)
    _native.call("mp_bfs_levels_host", n, indptr.ctypes.data, indices.ctypes.data, int(start), levels.ctypes.data,
                 queue.ctypes.data, tail.ctypes.data)
    return levels, queue, int(tail[0])


def heavy_edge_matching(indptr, indices, weights, node_weights, visit_order, max_cluster_weight):
    """``match[u]`` partner (or ``u``) of the visit-order heavy-edge greedy
    (numpy_impl.py:134-157)."""
    indptr, indices, weights = _i64(indptr), _i64(indices), _i64(weights)
    node_weights, visit_order = _i64(node_weights), _i64(visit_order)
    n = len(indptr) - 1
    match = np.empty(n, dtype=np.int64)
    if n:
        _native.call("mp_heavy_edge_matching", n, indptr.ctypes.data, indices.ctypes.data, weights.ctypes.data,
                     node_weights.ctypes.data, visit_order.ctypes.data, int(max_cluster_weight), match.ctypes.data)
    return match


def _inplace(a, name):
    if not (isinstance(a, np.ndarray) and a.dtype == np.int64 and a.flags.c_contiguous and a.flags.writeable):
        raise TypeError(f"{name} must be a writeable contiguous int64 array (it is updated in place)")
    return a


def refine_boundary_pass(indptr, indices, weights, assignment, block_weights, node_weights, cap, use_edge_weights):
    """One in-place boundary refinement sweep; returns the number of moves
    (numpy_impl.py:160-194).  ``assignment`` and ``block_weights`` change."""
    indptr, indices, weights, node_weights = _i64(indptr), _i64(indices), _i64(weights), _i64(node_weights)
    assignment = _inplace(assignment, "assignment")
    block_weights = _inplace(block_weights, "block_weights")
    n = len(indptr) - 1
    moves = np.zeros(1, dtype=np.int64)
    if n:
        _native.call("mp_refine_boundary_pass", n, indptr.ctypes.data, indices.ctypes.data, weights.ctypes.data,
                     assignment.ctypes.data, block_weights.ctypes.data, len(block_weights), node_weights.ctypes.data,
                     int(cap), int(bool(use_edge_weights)), moves.ctypes.data)
    return int(moves[0])


def cut_weight(indptr, indices, weights, assignment, use_edge_weights):
    """Total weight (or count) of edges across blocks (numpy_impl.py:197-206)."""
    indptr, indices, weights, assignment = _i64(indptr), _i64(indices), _i64(weights), _i64(assignment)
    n = len(indptr) - 1
    cut = np.zeros(1, dtype=np.int64)
    if n:
        _native.call("mp_cut_weight", n, indptr.ctypes.data, indices.ctypes.data, weights.ctypes.data,
                     assignment.ctypes.data, int(bool(use_edge_weights)), cut.ctypes.data)
    return int(cut[0])


def pairs_from_segments(seg_indptr, seg_values):
    """``(us, vs)``, every unordered pair inside each segment with ``us <
    vs``; pair order unspecified, as in the reference (numpy_impl.py:209-259)."""
    seg_indptr, seg_values = _i64(seg_indptr), _i64(seg_values)
    ns = len(seg_indptr) - 1
    total = np.zeros(1, dtype=np.int64)
    if ns <= 0:
        return np.empty(0, dtype=np.int64), np.empty(0, dtype=np.int64)
    _native.call("mp_pairs_from_segments", ns, seg_indptr.ctypes.data, seg_values.ctypes.data, None, None,
                 total.ctypes.data)
    us = np.empty(int(total[0]), dtype=np.int64)
    vs = np.empty(int(total[0]), dtype=np.int64)
    _native.call("mp_pairs_from_segments", ns, seg_indptr.ctypes.data, seg_values.ctypes.data, us.ctypes.data,
                 vs.ctypes.data, total.ctypes.data)
    return us, vs

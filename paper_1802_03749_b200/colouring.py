"""Colour assignments and the colouring entry points of the public API.

``ColourAssignment`` and the relabel-by-load rule follow the reference
(pkg/src/meshplan/colouring.py:22-74).  The greedy passes themselves run in
the native library: least-loaded element / block colouring is sequential by
definition (each choice depends on the counts of every earlier item) and
runs as host C++ (``mp_greedy_colour_csr``); intra-block thread colouring is
independent per block and runs on the GPU, one warp per block
(``mp_plan_thread_colours``).
"""

from dataclasses import dataclass

import numpy as np

from . import _native

CHOOSERS = ("least-loaded", "first-fit")


@dataclass(frozen=True)
class ColourAssignment:
    colours: np.ndarray
    num_colours: int
    counts: np.ndarray

    def __post_init__(self):
        for name in ("colours", "counts"):
            a = np.ascontiguousarray(getattr(self, name), dtype=np.int64)
            a.setflags(write=False)
            object.__setattr__(self, name, a)

    @classmethod
    def from_colours(cls, colours) -> "ColourAssignment":
        c = np.asarray(colours, dtype=np.int64)
        k = int(c.max()) + 1 if c.size else 0
        return cls(c, k, np.bincount(c, minlength=k))


def relabel_by_load(colours: np.ndarray, num: int) -> ColourAssignment:
    """Colour ids renumbered by descending item count, ties by old id."""
    counts = np.bincount(colours, minlength=num)
    rank = np.lexsort((np.arange(num), -counts))
    new_id = np.empty(num, dtype=np.int64)
    new_id[rank] = np.arange(num, dtype=np.int64)
    return ColourAssignment(new_id[colours], num, counts[rank])


def greedy_colour_csr(indptr, indices, n_points: int, least_loaded: bool) -> np.ndarray:
    """Native twin of ``_accel.greedy_colour_csr`` (numpy_impl.py:12-60)."""
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    n = len(indptr) - 1
    out = np.full(max(n, 0), -1, dtype=np.int64)
    if n > 0:
        _native.call("mp_greedy_colour_csr", n, indptr.ctypes.data, indices.ctypes.data, int(n_points),
                     int(bool(least_loaded)), out.ctypes.data)
    return out


def greedy_colour_adj(indptr, indices, order, least_loaded: bool) -> np.ndarray:
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    order = np.ascontiguousarray(order, dtype=np.int64)
    n = len(indptr) - 1
    out = np.full(max(n, 0), -1, dtype=np.int64)
    if n > 0:
        _native.call("mp_greedy_colour_adj", n, indptr.ctypes.data, indices.ctypes.data, order.ctypes.data,
                     int(bool(least_loaded)), out.ctypes.data)
    return out


def smallest_last_order(indptr, indices) -> np.ndarray:
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    n = len(indptr) - 1
    out = np.empty(max(n, 0), dtype=np.int64)
    if n > 0:
        _native.call("mp_smallest_last_order", n, indptr.ctypes.data, indices.ctypes.data, out.ctypes.data)
    return out


def colour_csr_least_loaded(indptr, indices, n_points: int) -> ColourAssignment:
    """Greedy least-loaded colouring + relabel (plan.py:232-257)."""
    c = greedy_colour_csr(indptr, indices, n_points, True)
    if c.size == 0:
        return ColourAssignment(c, 0, np.empty(0, dtype=np.int64))
    return relabel_by_load(c, int(c.max()) + 1)


def sort_threads_by_colour(colours: ColourAssignment):
    from .permutation import Permutation

    return Permutation.from_order(np.argsort(colours.colours, kind="stable").astype(np.int64))

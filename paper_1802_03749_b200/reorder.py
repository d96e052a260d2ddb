"""Point and element renumberings: the reference's ``meshplan.reorder`` API
(pkg/src/meshplan/reorder.py), computed on the GPU.

The plan builder calls the device forms directly on resident tensors
(``gpuplan.point_graph`` / ``gps_forward_graph`` / ``lex_order``,
``kway.writer_set_forward``); these are the public host-array entry points
with the reference's names, signatures and results, so a ``meshplan``
caller that renumbers a mesh itself finds them here:

==============================  ===================  ===============================
function                        reference            device work
==============================  ===================  ===============================
mesh_to_graph                   reorder.py:63-79     per-row clique pairs, sort/unique
bandwidth                       reorder.py:82-92     one max-reduction
gps_renumber                    reorder.py:115-141   level-synchronous BFS + LSD sorts
gps_levels                      reorder.py:144-158   BFS per component
lex_sort_elements               reorder.py:161-171   stable LSD sorts
reorder_points_by_writer_sets   reorder.py:174-203   padded-tuple LSD sorts
first_touch_renumber            reorder.py:206-217   first-position scatter-min + sort
==============================  ===================  ===============================

``PointGraph`` is the reference's CSR value type (symmetric, sorted, no
self-loops); ``from_edges`` builds it from host endpoint arrays as the
reference does.  Every function needs the GPU (no CPU execution path).
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _native, gpuplan
from .mesh import Mapping
from .permutation import Permutation


@dataclass(frozen=True)
class PointGraph:
    """Undirected CSR graph: symmetric, sorted neighbour lists, no self-loops."""

    n: int
    indptr: np.ndarray
    indices: np.ndarray

    def __post_init__(self):
        for name in ("indptr", "indices"):
            a = np.ascontiguousarray(getattr(self, name), dtype=np.int64)
            a.setflags(write=False)
            object.__setattr__(self, name, a)

    @classmethod
    def from_edges(cls, n: int, us, vs) -> "PointGraph":
        """CSR of the symmetric closure of the endpoint pairs; duplicate
        pairs and self-loops dropped (reorder.py:34-50)."""
        us = np.asarray(us, dtype=np.int64).ravel()
        vs = np.asarray(vs, dtype=np.int64).ravel()
        if n == 0:
            return cls(0, np.zeros(1, dtype=np.int64), np.empty(0, dtype=np.int64))
        off = us != vs
        both = np.unique(np.concatenate([us[off] * n + vs[off], vs[off] * n + us[off]]))
        src, dst = np.divmod(both, n)
        indptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(src, minlength=n), out=indptr[1:])
        return cls(n, indptr, dst)

    @property
    def num_edges(self) -> int:
        return len(self.indices) // 2

    def degrees(self) -> np.ndarray:
        return np.diff(self.indptr)

    def neighbours(self, u: int) -> np.ndarray:
        return self.indices[self.indptr[u]: self.indptr[u + 1]]


def _dev():
    _native.require_cuda()
    return torch.device("cuda")


def _table_d(m: Mapping) -> torch.Tensor:
    return gpuplan.upload(np.ascontiguousarray(m.table), _dev()).reshape(m.table.shape)


def _graph_d(g: PointGraph):
    dev = _dev()
    return (gpuplan.upload(g.indptr, dev), gpuplan.upload(g.indices, dev).to(torch.int32))


def _perm_from_fwd(fwd: torch.Tensor) -> Permutation:
    f = fwd.to(torch.int64)
    inv = torch.empty_like(f)
    inv[f] = torch.arange(f.numel(), device=f.device)
    return Permutation.unchecked(f.cpu().numpy(), inv.cpu().numpy())


def _perm_from_order(order: torch.Tensor) -> Permutation:
    o = order.to(torch.int64)
    fwd = torch.empty_like(o)
    fwd[o] = torch.arange(o.numel(), device=o.device)
    return Permutation.unchecked(fwd.cpu().numpy(), o.cpu().numpy())


def mesh_to_graph(m: Mapping) -> PointGraph:
    """Point-connectivity graph: the union over elements of the clique on
    each row's distinct points (reorder.py:63-79)."""
    n, arity = m.table.shape
    if n == 0 or arity < 2 or m.to_set.size == 0:
        return PointGraph.from_edges(m.to_set.size, [], [])
    indptr, indices = gpuplan.point_graph(_table_d(m), m.to_set.size)
    return PointGraph(m.to_set.size, indptr.cpu().numpy(), indices.to(torch.int64).cpu().numpy())


def bandwidth(g: PointGraph, perm: Permutation | None = None) -> int:
    """max |sigma(u) - sigma(v)| over the edges, 0 without edges (reorder.py:82-92)."""
    if len(g.indices) == 0:
        return 0
    indptr, indices = _graph_d(g)
    rows = torch.repeat_interleave(torch.arange(g.n, device=indptr.device), indptr[1:] - indptr[:-1])
    cols = indices.long()
    if perm is not None:
        f = gpuplan.upload(perm.forward, indptr.device)
        rows, cols = f[rows], f[cols]
    return int((rows - cols).abs().max())


def gps_renumber(g: PointGraph) -> Permutation:
    """Level-structure renumbering (reorder.py:115-141): components in order
    of their lowest index, each numbered by BFS level from a pseudo-peripheral
    root, within a level by (degree, index).  ``forward[old] = new``."""
    if g.n == 0:
        return Permutation.identity(0)
    indptr, indices = _graph_d(g)
    return _perm_from_fwd(gpuplan.gps_forward_graph(indptr, indices, g.n))


def gps_levels(g: PointGraph, perm: Permutation) -> np.ndarray:
    """Per-node BFS levels implied by a level-contiguous numbering: BFS from
    the first node (in the new numbering) of each component (reorder.py:144-158)."""
    levels = np.full(g.n, -1, dtype=np.int64)
    if g.n == 0:
        return levels
    indptr, indices = _graph_d(g)
    lv = torch.empty(g.n, dtype=torch.int32, device=indptr.device)
    done = torch.zeros(g.n, dtype=torch.bool, device=indptr.device)
    out = torch.full((g.n,), -1, dtype=torch.int64, device=indptr.device)
    inv = gpuplan.upload(perm.inverse, indptr.device)
    while True:
        pending = torch.nonzero(~done[inv])  # new positions whose node is unlevelled
        if pending.numel() == 0:
            break
        start = int(inv[int(pending[0, 0])])
        gpuplan.bfs(indptr, indices, start, lv)
        reached = lv >= 0
        out[reached] = lv[reached].long()
        done |= reached
    levels[:] = out.cpu().numpy()
    return levels


def lex_sort_elements(m: Mapping, point_perm: Permutation) -> Permutation:
    """Elements ordered by the sorted tuple of their renumbered points,
    stable for equal tuples (reorder.py:161-171)."""
    if m.table.shape[0] == 0:
        return Permutation.identity(0)
    fwd = gpuplan.upload(point_perm.forward, _dev())
    return _perm_from_order(gpuplan.lex_order(_table_d(m), fwd, max(m.to_set.size, 1)))


def reorder_points_by_writer_sets(m: Mapping, assignment) -> Permutation:
    """Points keyed by (number of distinct referencing blocks, the sorted
    block tuple, index) (reorder.py:174-203)."""
    from .kway import writer_set_forward

    npts = m.to_set.size
    if m.table.size == 0:
        return Permutation.identity(npts)
    a = gpuplan.upload(np.ascontiguousarray(assignment, dtype=np.int64), _dev())
    return _perm_from_fwd(writer_set_forward(_table_d(m), npts, a))


def first_touch_renumber(m: Mapping, elem_perm: Permutation) -> Permutation:
    """To-set points numbered by first appearance when the elements are
    visited in their new order; untouched points keep their relative order at
    the end (reorder.py:206-217)."""
    npts = m.to_set.size
    dev = _dev()
    if npts == 0:
        return Permutation.identity(0)
    flat = _table_d(m)[gpuplan.upload(elem_perm.inverse, dev)].reshape(-1).long()
    big = torch.iinfo(torch.int64).max
    first = torch.full((npts,), big, dtype=torch.int64, device=dev)
    if flat.numel():
        first.scatter_reduce_(0, flat, torch.arange(flat.numel(), device=dev), reduce="amin")
    # touched points by first position, then untouched ones by index
    key = torch.where(first == big, flat.numel() + torch.arange(npts, device=dev), first)
    return _perm_from_order(torch.argsort(key))

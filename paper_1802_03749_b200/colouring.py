"""Colour assignments and the colouring entry points of the public API.

``ColourAssignment`` and the relabel-by-load rule follow the reference
(pkg/src/meshplan/colouring.py:22-74).  The greedy passes themselves run in
the native library: least-loaded element / block colouring is sequential by
definition (each choice depends on the counts of every earlier item) and
runs as host C++ (``mp_greedy_colour_csr``); intra-block thread colouring is
independent per block and runs on the GPU, one warp per block
(``mp_plan_thread_colours``).

Public entry points with the reference's names and results
(colouring.py:43-176): ``colour_global`` and ``colour_blocks`` run the
greedy on the GPU (``mp_plan_block_colours``: lower-id conflict lists by
sorts, then one warp walks the items in order), ``colour_threads_in_block``
runs the per-block GPU kernel (first-fit, up to 1024 elements; the
least-loaded chooser or larger blocks take the native host twins of
``smallest_last_order`` / ``greedy_colour_adj``), ``block_conflict_graph``
is built on the GPU with sorts.
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


# ---- public colouring API (colouring.py:43-176) ----------------------------------


def normalize_slots(arity: int, written_slots=None) -> tuple:
    """None = every slot; accepts slot indices or a per-slot bool mask
    (colouring.py:43-53)."""
    if written_slots is None:
        return tuple(range(arity))
    written_slots = list(written_slots)
    if len(written_slots) == arity and all(isinstance(s, (bool, np.bool_)) for s in written_slots):
        return tuple(i for i, flag in enumerate(written_slots) if flag)
    slots = tuple(sorted(int(s) for s in written_slots))
    if any(s < 0 or s >= arity for s in slots):
        raise ValueError(f"written slots {slots} out of range for arity {arity}")
    return slots


def _check_chooser(chooser: str) -> None:
    if chooser not in CHOOSERS:
        raise ValueError(f"unknown colour chooser {chooser!r}; expected one of {CHOOSERS}")


def written_points_csr(m, written_slots=None, elements=None):
    """Per-element distinct written points as a host CSR (colouring.py:77-81)."""
    slots = normalize_slots(m.arity, written_slots)
    table = m.table if elements is None else m.table[np.asarray(elements, dtype=np.int64)]
    rows = np.sort(table[:, list(slots)], axis=1)
    if rows.size == 0:
        return np.zeros(len(rows) + 1, dtype=np.int64), np.empty(0, dtype=np.int64)
    keep = np.ones_like(rows, dtype=bool)
    keep[:, 1:] = rows[:, 1:] != rows[:, :-1]
    indptr = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(keep.sum(axis=1), out=indptr[1:])
    return indptr, rows[keep].astype(np.int64)


def _device_greedy(ptr_d, ids_d, chooser: str) -> ColourAssignment:
    import torch

    from . import gpuplan

    col, num, counts = gpuplan.colour_blocks_device(ptr_d.to(torch.int32), ids_d.to(torch.int32),
                                                    least_loaded=chooser == "least-loaded")
    return ColourAssignment(col.cpu().numpy(), num, counts)


def colour_global(m, written_slots=None, chooser: str = "least-loaded") -> ColourAssignment:
    """Greedy element colouring in element order; least-loaded colours are
    renumbered by descending load (colouring.py:84-99).  On the GPU."""
    import torch

    _check_chooser(chooser)
    _native.require_cuda()
    indptr, indices = written_points_csr(m, written_slots)
    if len(indptr) == 1:
        e = np.empty(0, dtype=np.int64)
        return ColourAssignment(e, 0, e.copy())
    return _device_greedy(torch.as_tensor(indptr, device="cuda"), torch.as_tensor(indices, device="cuda"), chooser)


def colour_blocks(part, m, written_slots=None, chooser: str = "least-loaded") -> ColourAssignment:
    """Blocks coloured so equal colours write disjoint points, blocks visited
    in id order over their distinct written points (colouring.py:102-124).
    The (block, point) pairs are deduplicated and grouped on the GPU."""
    import torch

    _check_chooser(chooser)
    slots = normalize_slots(m.arity, written_slots)
    n = m.table.shape[0]
    if len(part.assignment) != n:
        raise ValueError("partition does not cover the mapping's from-set")
    if part.num_blocks == 0:
        e = np.empty(0, dtype=np.int64)
        return ColourAssignment(e, 0, e.copy())
    _native.require_cuda()
    span = max(m.to_set.size, 1)
    tab = torch.as_tensor(np.ascontiguousarray(m.table[:, list(slots)]), device="cuda").long()
    blk = torch.as_tensor(np.asarray(part.assignment, dtype=np.int64), device="cuda")
    pairs = torch.unique(blk.repeat_interleave(len(slots)) * span + tab.reshape(-1))
    pb = torch.div(pairs, span, rounding_mode="floor")
    indptr = torch.zeros(part.num_blocks + 1, dtype=torch.int64, device="cuda")
    indptr[1:] = torch.cumsum(torch.bincount(pb, minlength=part.num_blocks), 0)
    return _device_greedy(indptr, pairs - pb * span, chooser)


def block_conflict_graph(block, m, written_slots=None):
    """Symmetric CSR of the block's elements that write a common point, local
    ids, sorted neighbour lists (colouring.py:127-149); built on the GPU."""
    import torch

    from .kway import _segment_pairs

    block = np.asarray(block, dtype=np.int64)
    k = len(block)
    indptr, points = written_points_csr(m, written_slots, elements=block)
    if k == 0 or points.size == 0:
        return np.zeros(k + 1, dtype=np.int64), np.empty(0, dtype=np.int64)
    _native.require_cuda()
    dev = torch.device("cuda")
    pts = torch.as_tensor(points, device=dev)
    owners = torch.repeat_interleave(torch.arange(k, device=dev), torch.as_tensor(np.diff(indptr), device=dev))
    keys, _ = torch.sort(pts * k + owners)  # grouped by point, owners ascending
    gp = torch.div(keys, k, rounding_mode="floor")
    own = keys - gp * k
    _, counts = torch.unique_consecutive(gp, return_counts=True)
    seg = torch.zeros(counts.numel() + 1, dtype=torch.int64, device=dev)
    seg[1:] = torch.cumsum(counts, 0)
    us, vs = _segment_pairs(seg, own)
    if us.numel():
        e = torch.unique(us * k + vs)
        us, vs = torch.div(e, k, rounding_mode="floor"), e % k
    src, dst = torch.cat([us, vs]), torch.cat([vs, us])
    order = torch.argsort(src * k + dst)
    src, dst = src[order], dst[order]
    adj = torch.zeros(k + 1, dtype=torch.int64, device=dev)
    adj[1:] = torch.cumsum(torch.bincount(src, minlength=k), 0)
    return adj.cpu().numpy(), dst.cpu().numpy()


def colour_threads_in_block(block, m, written_slots=None, chooser: str = "first-fit") -> ColourAssignment:
    """Greedy colouring of a block's elements over the smallest-last order of
    their conflict graph (colouring.py:152-166).  First-fit blocks of up to
    1024 elements run the planner's GPU kernel (one warp, bit-matrix conflict
    graph); the least-loaded chooser and larger blocks run the native host
    twins of the reference's sequential order and greedy."""
    import torch

    _check_chooser(chooser)
    block = np.asarray(block, dtype=np.int64)
    k = len(block)
    if k == 0:
        raise ValueError("block is empty")
    slots = normalize_slots(m.arity, written_slots)
    if chooser == "first-fit" and k <= 1024:
        from . import gpuplan

        _native.require_cuda()
        sub = torch.as_tensor(np.ascontiguousarray(m.table[block]), device="cuda").to(torch.int32)
        mask = 0
        for s_ in slots:
            mask |= 1 << s_
        bo = torch.tensor([0, k], dtype=torch.int32, device="cuda")
        cols, _, _ = gpuplan.thread_colours(bo, sub, mask, k)
        return ColourAssignment.from_colours(cols.cpu().numpy())
    adj_ptr, adj = block_conflict_graph(block, m, written_slots)
    order = smallest_last_order(adj_ptr, adj)
    return ColourAssignment.from_colours(greedy_colour_adj(adj_ptr, adj, order, chooser == "least-loaded"))

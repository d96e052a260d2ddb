"""Multilevel k-way partitioning of the iteration set (the ``partition`` reorder).

Bit-exact with the reference partitioner (pkg/src/meshplan/partition.py:47-350)
and its point reordering (reorder.py:174-203):

* thread graph G_M (elements adjacent when they share a point, weight =
  distinct shared points) -- GPU (sort / unique / segment pairs);
* coarsening: the reference's numpy PCG64 visit orders (drawn here with the
  same ``np.random.default_rng(seed)`` calls, level by level), heavy-edge
  matching and contraction on the GPU (the matching in dependency rounds that
  reproduce the sequential greedy; MESHPLAN_HOST_MATCHING=1 runs the native
  host sweep instead);
* recursive region-growing bisection, rebalancing and boundary-refinement
  sweeps -- native host C++ (inherently sequential, in-place sweeps);
* writer-set point order -- GPU stable LSD sorts over padded block tuples.
"""

import math
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .errors import MeshValidationError
from .partition import Partition, PartitionConfig, compute_effective_block_size


@dataclass(frozen=True)
class ThreadGraph:
    n: int
    indptr: np.ndarray
    indices: np.ndarray
    weights: np.ndarray
    device: tuple = field(default=None, compare=False, repr=False)  # device (indptr, indices, weights), if built there

    @property
    def num_edges(self) -> int:
        return len(self.indices) // 2


def _segment_pairs(seg_ptr: torch.Tensor, vals: torch.Tensor):
    """All (min, max) pairs inside each segment (pairs_from_segments,
    numpy_impl.py:209-259), batched by segment length."""
    lengths = seg_ptr[1:] - seg_ptr[:-1]
    us, vs = [], []
    for k in torch.unique(lengths).tolist():
        if k < 2:
            continue
        starts = seg_ptr[:-1][lengths == k]
        block = vals[starts[:, None] + torch.arange(k, device=vals.device)]
        ia, ib = torch.triu_indices(k, k, 1, device=vals.device)
        a, b = block[:, ia].reshape(-1), block[:, ib].reshape(-1)
        us.append(torch.minimum(a, b))
        vs.append(torch.maximum(a, b))
    if not us:
        e = torch.empty(0, dtype=torch.long, device=vals.device)
        return e, e.clone()
    return torch.cat(us), torch.cat(vs)


def thread_graph_device(map_d: torch.Tensor, npts: int):
    """G_M of one mapping (partition.py:47-95) as device tensors."""
    n, ar = map_d.shape
    dev = map_d.device
    pts = map_d.long().reshape(-1)
    el = torch.arange(n, device=dev).repeat_interleave(ar)
    refs = torch.unique(pts * n + el) if n else pts
    rp = torch.div(refs, max(n, 1), rounding_mode="floor")
    re = refs - rp * n
    seg = torch.zeros(npts + 1, dtype=torch.long, device=dev)
    if refs.numel():
        seg[1:] = torch.cumsum(torch.bincount(rp, minlength=npts), 0)
    us, vs = _segment_pairs(seg, re)
    if us.numel():
        keys, w = torch.unique(us * n + vs, return_counts=True)
        us = torch.div(keys, n, rounding_mode="floor")
        vs = keys - us * n
    else:
        w = us.clone()
    src = torch.cat([us, vs])
    dst = torch.cat([vs, us])
    ww = torch.cat([w, w])
    order = torch.argsort(src * max(n, 1) + dst)
    src, dst, ww = src[order], dst[order], ww[order]
    indptr = torch.zeros(n + 1, dtype=torch.long, device=dev)
    if src.numel():
        indptr[1:] = torch.cumsum(torch.bincount(src, minlength=n), 0)
    return indptr, dst, ww


def build_thread_graph(mappings) -> ThreadGraph:
    """Public twin of partition.build_thread_graph for single-to-set loops."""
    if not mappings:
        raise ValueError("need at least one mapping")
    m = mappings[0]
    if any(x.from_set is not m.from_set for x in mappings):
        raise ValueError("all mappings must share the same from-set")
    if len(mappings) > 1:
        raise MeshValidationError("the device partitioner takes one mapping per loop")
    _native.require_cuda()
    map_d = torch.as_tensor(np.ascontiguousarray(m.table), device="cuda")
    ip, ix, w = thread_graph_device(map_d, m.to_set.size)
    return ThreadGraph(m.from_set.size, ip.cpu().numpy(), ix.cpu().numpy(), w.cpu().numpy())


def _contract(ip, ix, ew, nw, mt):
    """partition._contract (173-195) on device tensors; returns device tensors
    (indptr, indices, weights, node_w, cmap) of the coarse graph."""
    dev = ip.device
    n = nw.numel()
    rep = torch.minimum(torch.arange(n, device=dev), mt)
    reps = torch.unique(rep)
    cid = torch.empty(n, dtype=torch.long, device=dev)
    cid[reps] = torch.arange(reps.numel(), device=dev)
    cmap = cid[rep]
    nc = reps.numel()
    cw = torch.bincount(cmap, weights=nw.double(), minlength=nc).long()
    rows = cmap.repeat_interleave(ip[1:] - ip[:-1])
    cols = cmap[ix]
    keep = rows != cols
    rows, cols, ew = rows[keep], cols[keep], ew[keep]
    uniq, inv = torch.unique(rows * nc + cols, return_inverse=True)
    summed = torch.bincount(inv, weights=ew.double(), minlength=uniq.numel()).long()
    r = torch.div(uniq, nc, rounding_mode="floor")
    c = uniq - r * nc
    cip = torch.zeros(nc + 1, dtype=torch.long, device=dev)
    if r.numel():
        cip[1:] = torch.cumsum(torch.bincount(r, minlength=nc), 0)
    return cip, c, summed, cw, cmap


def _match_device(ip, ix, ew, nw, visit: np.ndarray, max_cluster: int) -> torch.Tensor:
    """_accel.heavy_edge_matching (partition.py:317) on the GPU, in dependency
    rounds (mp_heavy_edge_matching_device); equal to the sequential greedy."""
    n = nw.numel()
    vis = torch.as_tensor(visit, device=ip.device)
    match = torch.empty(n, dtype=torch.long, device=ip.device)
    rounds = np.zeros(1, dtype=np.int32)
    _native.call("mp_heavy_edge_matching_device", n, _native.ptr(ip), _native.ptr(ix), _native.ptr(ew),
                 _native.ptr(nw), _native.ptr(vis), int(max_cluster), _native.ptr(match), rounds.ctypes.data,
                 torch.cuda.current_stream().cuda_stream)
    return match


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def partition_kway(g: ThreadGraph, cfg: PartitionConfig) -> Partition:
    """partition.partition_kway (288-350), bit-exact."""
    eff_size, eff_tol = compute_effective_block_size(cfg)
    n = g.n
    if n == 0:
        return Partition(np.empty(0, dtype=np.int64), 0, cut=0)
    nb = -(-n // eff_size)
    use_w = int(not cfg.unweighted_cut)
    if nb == 1:
        return Partition(np.zeros(n, dtype=np.int64), 1, cut=0)
    cap = min(cfg.block_size, max(int(math.floor(eff_tol * n / nb)), -(-n // nb)))
    indptr = np.ascontiguousarray(g.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(g.indices, dtype=np.int64)
    weights = np.ascontiguousarray(g.weights, dtype=np.int64)
    node_w = np.ones(n, dtype=np.int64)
    rng = np.random.default_rng(cfg.seed)
    target = max(2 * nb, 64)
    max_cluster = max(1, cap // 4)
    levels = []
    timing = os.environ.get("MESHPLAN_KWAY_TIMING")
    t0 = time.perf_counter()
    tick = (lambda what: print(f"[kway] {what}: {time.perf_counter() - t0:.2f}s", flush=True)) if timing else (lambda what: None)
    host_match = bool(os.environ.get("MESHPLAN_HOST_MATCHING"))
    h = lambda x: x.cpu().numpy().astype(np.int64)  # noqa: E731
    if g.device is not None:
        gd = tuple(t.long() for t in g.device)
    else:
        gd = tuple(torch.as_tensor(a, device="cuda") for a in (indptr, indices, weights))
    nw_d = torch.ones(n, dtype=torch.long, device=gd[0].device)
    while len(node_w) > target:
        visit = rng.permutation(len(node_w)).astype(np.int64)
        tick(f"  visit order ({len(node_w)} nodes)")
        if host_match:
            match = np.empty(len(node_w), dtype=np.int64)
            _native.call("mp_heavy_edge_matching", len(node_w), _p(indptr), _p(indices), _p(weights), _p(node_w),
                         _p(visit), max_cluster, _p(match))
            match_d = torch.as_tensor(match, device=gd[0].device)
        else:
            match_d = _match_device(*gd, nw_d, visit, max_cluster)
        tick("  matching")
        cip_d, cix_d, cw_d, cnw_d, cmap_d = _contract(*gd, nw_d, match_d)
        tick("  contraction")
        if cnw_d.numel() >= 0.95 * len(node_w):
            break
        levels.append((indptr, indices, weights, node_w, h(cmap_d)))
        gd, nw_d = (cip_d, cix_d, cw_d), cnw_d
        indptr, indices, weights, node_w = h(cip_d), h(cix_d), h(cw_d), h(cnw_d)
    tick(f"coarsening ({len(levels)} levels, coarsest {len(node_w)} nodes)")
    assignment = np.empty(len(node_w), dtype=np.int64)
    _native.call("mp_initial_partition", len(node_w), _p(indptr), _p(indices), _p(node_w), nb, cap, _p(assignment))
    tick("initial partition")

    def refine(ip, ix, w, a, nw):
        bw = np.bincount(a, weights=nw, minlength=nb).astype(np.int64)
        _native.call("mp_rebalance", len(nw), _p(ip), _p(ix), _p(w), _p(a), _p(bw), nb, _p(nw), cap, use_w)
        tick("    rebalance")
        # The reference asserts the cut never rises around each pass
        # (partition.py:329-336).  A pass moves a node only for a strictly
        # positive gain (numpy_impl.py:160-194: best_gain starts at 0, ties only
        # between positive gains), and each move lowers the cut by its gain, so
        # the assertion cannot fire; the two O(E) cut sweeps per pass are skipped
        # (MESHPLAN_KWAY_CHECK=1 re-enables them).
        check = bool(os.environ.get("MESHPLAN_KWAY_CHECK"))
        cut = np.zeros(1, dtype=np.int64)
        moves = np.zeros(1, dtype=np.int64)
        if not check:  # the 8 sweeps in one call, later sweeps over the changed frontier only
            _native.call("mp_refine_boundary", len(nw), _p(ip), _p(ix), _p(w), _p(a), _p(bw), nb, _p(nw), cap,
                         use_w, 8, _p(moves))
            return
        for _ in range(8):
            if check:
                _native.call("mp_cut_weight", len(nw), _p(ip), _p(ix), _p(w), _p(a), use_w, _p(cut))
                before = int(cut[0])
            _native.call("mp_refine_boundary_pass", len(nw), _p(ip), _p(ix), _p(w), _p(a), _p(bw), nb, _p(nw), cap,
                         use_w, _p(moves))
            if check:
                _native.call("mp_cut_weight", len(nw), _p(ip), _p(ix), _p(w), _p(a), use_w, _p(cut))
                if int(cut[0]) > before:
                    raise AssertionError(f"refinement increased cut: {before} -> {int(cut[0])}")
            if int(moves[0]) == 0:
                break

    refine(indptr, indices, weights, assignment, node_w)
    tick("refine coarsest")
    for fip, fix, fw, fnw, cmap in reversed(levels):
        assignment = np.ascontiguousarray(assignment[cmap])
        tick("    projection")
        indptr, indices, weights, node_w = fip, fix, fw, fnw
        refine(indptr, indices, weights, assignment, node_w)
        tick(f"refine level with {len(fnw)} nodes")
    cut = np.zeros(1, dtype=np.int64)
    gi, gx, gw = (np.ascontiguousarray(a, dtype=np.int64) for a in (g.indptr, g.indices, g.weights))
    _native.call("mp_cut_weight", n, _p(gi), _p(gx), _p(gw), _p(assignment), use_w, _p(cut))
    part = Partition(assignment, nb, cut=int(cut[0]))
    if part.imbalance() > eff_tol + 1e-12 or int(part.block_sizes().max()) > cfg.block_size:
        part = Partition(assignment, nb, over_tolerance=True, cut=int(cut[0]))
    return part


def writer_set_forward(map_d: torch.Tensor, npts: int, assignment: torch.Tensor) -> torch.Tensor:
    """Forward point permutation of reorder_points_by_writer_sets (174-203):
    key (number of distinct writer blocks, sorted block tuple, id)."""
    dev = map_d.device
    n, ar = map_d.shape
    ids = torch.arange(npts, dtype=torch.long, device=dev)
    if n == 0:
        return ids
    span = int(assignment.max()) + 1
    pairs = torch.unique(map_d.long().reshape(-1) * span + assignment.repeat_interleave(ar))
    pp = torch.div(pairs, span, rounding_mode="floor")
    pb = pairs - pp * span
    cnt = torch.bincount(pp, minlength=npts)
    start = torch.zeros(npts + 1, dtype=torch.long, device=dev)
    start[1:] = torch.cumsum(cnt, 0)
    L = int(cnt.max())
    pad = torch.full((npts, max(L, 1)), -1, dtype=torch.long, device=dev)
    rank = torch.arange(pairs.numel(), device=dev) - start[pp]
    pad[pp, rank] = pb
    order = ids
    for col in range(L - 1, -1, -1):  # LSD: last tuple entry first, then count
        _, i = torch.sort(pad[order, col], stable=True)
        order = order[i]
    _, i = torch.sort(cnt[order], stable=True)
    order = order[i]
    fwd = torch.empty_like(order)
    fwd[order] = ids
    return fwd


@dataclass
class PlanPartition:
    order: torch.Tensor        # element order (old index at each new position)
    point_fwd: torch.Tensor    # forward point permutation
    block_sizes: np.ndarray
    meta: dict


def partition_for_plan(map_d: torch.Tensor, npts: int, config) -> PlanPartition:
    """The partition branch of plan._reorder_for_plan (plan.py:330-352)."""
    n = map_d.shape[0]
    ip, ix, w = thread_graph_device(map_d, npts)
    g = ThreadGraph(n, ip.cpu().numpy(), ix.cpu().numpy(), w.cpu().numpy(), device=(ip, ix, w))
    part = partition_kway(g, config.partition_config())
    a = torch.as_tensor(part.assignment, device=map_d.device)
    order = torch.as_tensor(np.argsort(part.assignment, kind="stable"), device=map_d.device)
    pf = writer_set_forward(map_d, npts, a)
    meta = {"num_blocks": part.num_blocks, "cut": part.cut, "over_tolerance": part.over_tolerance,
            "imbalance": part.imbalance()}
    return PlanPartition(order, pf, part.block_sizes(), meta)

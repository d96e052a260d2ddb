"""``reorder="cluster"``: a parallel GPU blocking (extension, not in the reference).

The reference ``partition`` mode (multilevel k-way, partition.py:288-350) is
reproduced bit for bit by :mod:`.kway`, but its sweeps are sequential by
definition, so at 64M elements it takes minutes.  This mode builds blocks of
the same kind -- compact element clusters of at most ``block_size``
elements, then writer-set point order (reorder.py:174-203) -- with a fully
parallel algorithm: repeated heavy-edge *handshake* matching on the element
graph G_M (each node proposes to its heaviest admissible neighbour, mutual
proposals merge; weights = shared points, so compact merges win) and GPU
contraction, until clusters stop growing.  Every cluster is one block.

It is deterministic (ties broken by a fixed hash of the node id) but not
equal to the reference partition, so plans built with it are judged by the
reference's own invariants (race freedom, block widths, staging coverage)
and by reuse / colour counts, not by plan bit-equality.
"""

import numpy as np
import torch

from .kway import thread_graph_device


def _hash32(x: torch.Tensor) -> torch.Tensor:
    mask = 0xFFFFFFFF
    x = (x * 2654435761) & mask
    x = x ^ (x >> 15)
    x = (x * 0x2C1B3C6D) & mask
    return x ^ (x >> 12)


def handshake_match(indptr, indices, weights, node_w, cap: int, rounds: int = 6) -> torch.Tensor:
    """Parallel heavy-edge matching: match[u] = v (pairs) or u (unmatched)."""
    dev = indptr.device
    n = node_w.numel()
    rows = torch.repeat_interleave(torch.arange(n, device=dev), indptr[1:] - indptr[:-1])
    match = torch.full((n,), -1, dtype=torch.long, device=dev)
    prio = _hash32(indices) & 0xFFFF
    base = (weights.clamp(max=2**14) << 48) | (prio << 32) | indices  # heaviest, then hash, then id
    ids = torch.arange(n, device=dev)
    for _ in range(rounds):
        ok = (match[rows] < 0) & (match[indices] < 0) & (rows != indices) & (node_w[rows] + node_w[indices] <= cap)
        if not bool(ok.any()):
            break
        key = torch.where(ok, base, torch.full_like(base, -1))
        best_key = torch.full((n,), -1, dtype=torch.long, device=dev).scatter_reduce(0, rows, key, "amax")
        best = torch.where(best_key >= 0, best_key & 0xFFFFFFFF, torch.full_like(best_key, -1))
        safe = best.clamp(min=0)
        mutual = (best >= 0) & (best[safe] == ids) & (match < 0)
        match = torch.where(mutual, best, match)
    return torch.where(match < 0, ids, match)


def contract_device(indptr, indices, weights, node_w, match):
    """Collapse matched pairs (same rule as partition._contract, on the GPU)."""
    dev = indptr.device
    n = node_w.numel()
    rep = torch.minimum(torch.arange(n, device=dev), match)
    reps, cmap = torch.unique(rep, return_inverse=True)
    nc = reps.numel()
    cw = torch.zeros(nc, dtype=torch.long, device=dev).index_add_(0, cmap, node_w)
    r = cmap.repeat_interleave(indptr[1:] - indptr[:-1])
    c = cmap[indices]
    keep = r != c
    r, c, w = r[keep], c[keep], weights[keep]
    uniq, inv = torch.unique(r * nc + c, return_inverse=True)
    sw = torch.zeros(uniq.numel(), dtype=torch.long, device=dev).index_add_(0, inv, w)
    r = torch.div(uniq, nc, rounding_mode="floor")
    cip = torch.zeros(nc + 1, dtype=torch.long, device=dev)
    if r.numel():
        cip[1:] = torch.cumsum(torch.bincount(r, minlength=nc), 0)
    return cip, uniq - r * nc, sw, cw, cmap


def cluster_assignment(map_d: torch.Tensor, npts: int, block_size: int, max_levels: int = 24):
    """Cluster id per element (clusters of <= block_size elements)."""
    n = map_d.shape[0]
    dev = map_d.device
    ip, ix, w = thread_graph_device(map_d, npts)
    node_w = torch.ones(n, dtype=torch.long, device=dev)
    assign = torch.arange(n, dtype=torch.long, device=dev)
    for _ in range(max_levels):
        m = handshake_match(ip, ix, w, node_w, block_size)
        merged = int((m != torch.arange(m.numel(), device=dev)).sum())
        if merged < 0.02 * m.numel():
            break
        ip, ix, w, node_w, cmap = contract_device(ip, ix, w, node_w, m)
        assign = cmap[assign]
    return assign, int(node_w.numel())


def cluster_order(map_d: torch.Tensor, npts: int, block_size: int, gps_elem_rank: torch.Tensor | None = None):
    """(element order, block sizes, meta): clusters ordered by their first
    element in ``gps_elem_rank`` order (or id), elements within a cluster in
    that order too."""
    assign, ncl = cluster_assignment(map_d, npts, block_size)
    n = assign.numel()
    dev = assign.device
    rank = gps_elem_rank if gps_elem_rank is not None else torch.arange(n, device=dev)
    first = torch.full((ncl,), n, dtype=torch.long, device=dev).scatter_reduce(0, assign, rank, "amin")
    _, corder = torch.sort(first, stable=True)
    cid = torch.empty_like(corder)
    cid[corder] = torch.arange(ncl, device=dev)
    key = cid[assign] * (n + 1) + rank
    order = torch.argsort(key)
    sizes = torch.bincount(cid[assign], minlength=ncl).cpu().numpy()
    return order, cid[assign][order], sizes, {"num_blocks": int(ncl), "method": "gpu handshake clustering"}

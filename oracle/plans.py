"""Oracle plan builders (test infrastructure only -- see oracle/__init__.py).

Loop-for-loop restatements of the reference planner for single-mapping
loops.  Every function cites the reference code it restates.  Inputs are a
mapping ``table`` (n, arity) int64, the to-set size ``npts`` and the slot
lists the loop reads / writes.
"""

import math
from collections import deque

import numpy as np


# ---- _accel kernels (numpy_impl.py) ------------------------------------------------


def greedy_colour_csr(indptr, indices, n_points, least_loaded):
    """numpy_impl.py:12-60."""
    n = len(indptr) - 1
    colours = np.full(n, -1, dtype=np.int64)
    pcols = [[] for _ in range(n_points)]
    counts = []
    for i in range(n):
        forbidden = set()
        pts = indices[indptr[i]:indptr[i + 1]]
        for p in pts:
            forbidden.update(pcols[p])
        best = -1
        if least_loaded:
            best_count = None
            for c in range(len(counts)):
                if c not in forbidden and (best_count is None or counts[c] < best_count):
                    best, best_count = c, counts[c]
        else:
            for c in range(len(counts)):
                if c not in forbidden:
                    best = c
                    break
        if best < 0:
            best = len(counts)
            counts.append(0)
        colours[i] = best
        counts[best] += 1
        for p in pts:
            pcols[p].append(best)
    return colours


def greedy_colour_adj(indptr, indices, order, least_loaded=False):
    """numpy_impl.py:62-92."""
    n = len(indptr) - 1
    colours = np.full(n, -1, dtype=np.int64)
    counts = []
    for u in order:
        forbidden = {int(colours[v]) for v in indices[indptr[u]:indptr[u + 1]] if colours[v] >= 0}
        best = -1
        if least_loaded:
            best_count = None
            for c in range(len(counts)):
                if c not in forbidden and (best_count is None or counts[c] < best_count):
                    best, best_count = c, counts[c]
        else:
            for c in range(len(counts)):
                if c not in forbidden:
                    best = c
                    break
        if best < 0:
            best = len(counts)
            counts.append(0)
        colours[u] = best
        counts[best] += 1
    return colours


def smallest_last_order(indptr, indices):
    """numpy_impl.py:95-111: argmin of key = deg*(n+1)+u, neighbours decremented."""
    n = len(indptr) - 1
    key = np.diff(indptr).astype(np.int64) * (n + 1) + np.arange(n)
    removed = np.iinfo(np.int64).max
    order = np.empty(n, dtype=np.int64)
    for pos in range(n - 1, -1, -1):
        u = int(np.argmin(key))
        order[pos] = u
        key[u] = removed
        for v in indices[indptr[u]:indptr[u + 1]]:
            if key[v] != removed:
                key[v] -= n + 1
    return order


def bfs_levels(indptr, indices, start):
    """numpy_impl.py:114-131."""
    n = len(indptr) - 1
    levels = np.full(n, -1, dtype=np.int64)
    levels[start] = 0
    q = deque([start])
    seen = [start]
    while q:
        u = q.popleft()
        for v in indices[indptr[u]:indptr[u + 1]]:
            if levels[v] < 0:
                levels[v] = levels[u] + 1
                q.append(v)
                seen.append(v)
    return levels, np.asarray(seen, dtype=np.int64)


# ---- colouring helpers (colouring.py / plan.py) ------------------------------------


def dedup_rows(rows):
    """colouring.py:56-65."""
    if rows.size == 0:
        return np.zeros(len(rows) + 1, dtype=np.int64), np.empty(0, dtype=np.int64)
    srt = np.sort(rows, axis=1)
    keep = np.ones_like(srt, dtype=bool)
    keep[:, 1:] = srt[:, 1:] != srt[:, :-1]
    return np.concatenate(([0], np.cumsum(keep.sum(1)))).astype(np.int64), srt[keep].astype(np.int64)


def relabel_by_load(colours, num):
    """colouring.py:68-74."""
    counts = np.bincount(colours, minlength=num)
    rank = np.lexsort((np.arange(num), -counts))
    remap = np.empty(num, dtype=np.int64)
    remap[rank] = np.arange(num)
    return remap[colours], counts[rank]


def thread_colours_for_block(table_block_w):
    """plan.py:260-284 for one block: rows = its elements' written points."""
    k = table_block_w.shape[0]
    adj = [set() for _ in range(k)]
    by_point = {}
    for e in range(k):
        for p in set(table_block_w[e].tolist()):
            by_point.setdefault(p, []).append(e)
    for owners in by_point.values():
        for a in owners:
            for b in owners:
                if a != b:
                    adj[a].add(b)
    indptr = np.zeros(k + 1, dtype=np.int64)
    indptr[1:] = np.cumsum([len(s) for s in adj])
    indices = np.array([v for s in adj for v in sorted(s)], dtype=np.int64)
    if indices.size == 0:
        return np.zeros(k, dtype=np.int64)
    order = smallest_last_order(indptr, indices)
    return greedy_colour_adj(indptr, indices, order, False)


def split_oversized(offsets, limit):
    """plan.py:451-464."""
    out = [int(offsets[0])]
    for end in offsets[1:]:
        pending = [(out[-1], int(end))]
        while pending:
            lo, hi = pending.pop(0)
            if hi - lo > limit:
                mid = lo + (hi - lo + 1) // 2
                pending = [(lo, mid), (mid, hi)] + pending
            else:
                out.append(hi)
    return np.asarray(out, dtype=np.int64)


def block_point_lists(table_sel, block_offsets):
    """plan.py:582-603: ascending unique ids per block (CSR)."""
    nb = len(block_offsets) - 1
    parts = [np.unique(table_sel[block_offsets[b]:block_offsets[b + 1]]) for b in range(nb)]
    indptr = np.concatenate(([0], np.cumsum([p.size for p in parts]))).astype(np.int64)
    return indptr, (np.concatenate(parts).astype(np.int64) if parts else np.empty(0, dtype=np.int64))


# ---- reorderings (reorder.py) ---------------------------------------------------------


def point_graph(table, npts):
    """reorder.py:63-79 (clique union), adjacency as CSR."""
    adj = [set() for _ in range(npts)]
    for row in table:
        pts = sorted(set(int(v) for v in row))
        for a in pts:
            for b in pts:
                if a != b:
                    adj[a].add(b)
    indptr = np.concatenate(([0], np.cumsum([len(s) for s in adj]))).astype(np.int64)
    indices = np.array([v for s in adj for v in sorted(s)], dtype=np.int64)
    return indptr, indices


def gps_forward(table, npts):
    """reorder.py:95-141: forward point permutation."""
    indptr, indices = point_graph(table, npts)
    deg = np.diff(indptr)
    assigned = np.zeros(npts, dtype=bool)
    order = []
    for start in range(npts):
        if assigned[start]:
            continue
        _, comp = bfs_levels(indptr, indices, start)
        comp = np.sort(comp)
        assigned[comp] = True
        if comp.size == 1:
            order.append(comp)
            continue
        loc = comp[np.lexsort((comp, deg[comp]))]
        u = int(loc[0])
        lv, _ = bfs_levels(indptr, indices, u)
        ecc = int(lv[comp].max())
        while True:
            last = comp[lv[comp] == ecc]
            v = int(last[np.lexsort((last, deg[last]))][0])
            lv_v, _ = bfs_levels(indptr, indices, v)
            ecc_v = int(lv_v[comp].max())
            if ecc_v > ecc:
                u, lv, ecc = v, lv_v, ecc_v
            else:
                break
        levels, _ = bfs_levels(indptr, indices, u)
        order.append(comp[np.lexsort((comp, deg[comp], levels[comp]))])
    order = np.concatenate(order) if order else np.empty(0, dtype=np.int64)
    fwd = np.empty(npts, dtype=np.int64)
    fwd[order] = np.arange(npts)
    return fwd


def lex_order(table, point_fwd):
    """reorder.py:161-171."""
    if table.shape[0] == 0:
        return np.empty(0, dtype=np.int64)
    keys = np.sort(point_fwd[table], axis=1)
    return np.lexsort(tuple(keys[:, c] for c in range(keys.shape[1] - 1, -1, -1))).astype(np.int64)


# ---- plan builders --------------------------------------------------------------------


def _fwd_of_order(order):
    fwd = np.empty(len(order), dtype=np.int64)
    fwd[order] = np.arange(len(order))
    return fwd


def reorder(table, npts, mode):
    """Returns (table', elem_fwd, point_fwd) for none / gps (plan.py:320-329)."""
    n = table.shape[0]
    if mode == "none":
        return table, np.arange(n), np.arange(npts)
    if mode == "gps":
        pf = gps_forward(table, npts)
        order = lex_order(table, pf)
        return pf[table[order]], _fwd_of_order(order), pf
    raise ValueError(mode)


def global_plan(table, npts, wslots, mode="none"):
    """plan.py:408-448 (none/gps): returns dict of plan arrays."""
    t2, efwd, pfwd = reorder(table, npts, mode)
    indptr, idx = dedup_rows(t2[:, wslots])
    col = greedy_colour_csr(indptr, idx, max(npts, 1), True)
    n = t2.shape[0]
    if n:
        col, counts = relabel_by_load(col, int(col.max()) + 1)
        order = np.argsort(col, kind="stable")
        t2 = t2[order]
        efwd = _fwd_of_order(order)[efwd]
        col = col[order]
        offsets = np.concatenate(([0], np.cumsum(np.bincount(col)))).astype(np.int64)
    else:
        offsets = np.zeros(1, dtype=np.int64)
    return {"table": t2, "elem_fwd": efwd, "point_fwd": pfwd, "colours": col, "colour_offsets": offsets}


def hier_plan(table, npts, wslots, sslots, block_size, mode="none", sizes=None):
    """plan.py:467-579 for none/gps (chunking) or given block ``sizes``."""
    t2, efwd, pfwd = reorder(table, npts, mode)
    n = t2.shape[0]
    if sizes is None:
        offsets = np.append(np.arange(0, n, block_size), n) if n else np.zeros(1, dtype=np.int64)
    else:
        offsets = np.concatenate(([0], np.cumsum(sizes)))
    offsets = split_oversized(offsets, block_size)
    nb = len(offsets) - 1
    wp, wi = block_point_lists(t2[:, wslots], offsets)
    total = int(wi.max()) + 1 if wi.size else 1
    bc = greedy_colour_csr(wp, wi, total, True)
    nbc = int(bc.max()) + 1 if bc.size else 0
    if nbc:
        bc, _ = relabel_by_load(bc, nbc)
    tcol = np.zeros(n, dtype=np.int64)
    tcounts = np.zeros(nb, dtype=np.int64)
    order = np.arange(n)
    for b in range(nb):
        lo, hi = int(offsets[b]), int(offsets[b + 1])
        tc = thread_colours_for_block(t2[lo:hi][:, wslots])
        intra = np.argsort(tc, kind="stable")
        order[lo:hi] = lo + intra
        tcol[lo:hi] = tc[intra]
        tcounts[b] = tc.max() + 1 if tc.size else 0
    t2 = t2[order]
    efwd = _fwd_of_order(order)[efwd]
    sp, si = block_point_lists(t2[:, sslots], offsets)
    return {"table": t2, "elem_fwd": efwd, "point_fwd": pfwd, "block_offsets": offsets, "block_colours": bc,
            "num_block_colours": nbc, "thread_colours": tcol, "thread_colour_counts": tcounts,
            "staged": (sp, si), "written": (wp, wi)}


def effective_block_size(block_size, tolerance, epsilon):
    """partition.py:123-134 (Eq. 1-2)."""
    eff = int(math.floor(block_size / tolerance))
    return eff, (block_size + epsilon) / eff

"""Oracle k-way partitioner pieces (test infrastructure only -- see oracle/__init__.py).

Restates numpy_impl.py:134-206 (matching, refinement, cut) and
partition.py:198-285 (bisection seeding, rebalancing) loop for loop.
"""

import numpy as np


def heavy_edge_matching(indptr, indices, weights, node_w, visit, max_cluster):
    """numpy_impl.py:134-157."""
    match = np.full(len(indptr) - 1, -1, dtype=np.int64)
    for u in visit:
        if match[u] >= 0:
            continue
        best, best_w = u, -1
        for j in range(indptr[u], indptr[u + 1]):
            v = indices[j]
            if match[v] >= 0 or v == u or node_w[u] + node_w[v] > max_cluster:
                continue
            if weights[j] > best_w or (weights[j] == best_w and v < best):
                best, best_w = v, weights[j]
        match[u] = best
        if best != u:
            match[best] = u
    return match


def cut_weight(indptr, indices, weights, a, use_w):
    """numpy_impl.py:197-206."""
    total = 0
    for u in range(len(indptr) - 1):
        for j in range(indptr[u], indptr[u + 1]):
            v = indices[j]
            if u < v and a[u] != a[v]:
                total += weights[j] if use_w else 1
    return int(total)


def refine_boundary_pass(indptr, indices, weights, a, bw, node_w, cap, use_w):
    """numpy_impl.py:160-194 (mutates a, bw)."""
    moves = 0
    for u in range(len(indptr) - 1):
        own = a[u]
        conn = {}
        order = []
        for j in range(indptr[u], indptr[u + 1]):
            b = a[indices[j]]
            if b not in conn:
                conn[b] = 0
                order.append(b)
            conn[b] += weights[j] if use_w else 1
        best, best_gain = own, 0
        for b in order:
            if b == own:
                continue
            gain = conn[b] - conn.get(own, 0)
            if gain > best_gain or (gain == best_gain and best != own and b < best):
                if bw[b] + node_w[u] <= cap and bw[own] - node_w[u] > 0:
                    best, best_gain = b, gain
        if best != own:
            a[u] = best
            bw[own] -= node_w[u]
            bw[best] += node_w[u]
            moves += 1
    return moves


def grow_bisection(indptr, indices, node_w, subset, k1, k2, cap):
    """partition.py:198-236."""
    total = int(node_w[subset].sum())
    lower = max(0, total - k2 * cap)
    upper = min(k1 * cap, total)
    target = min(max(int(round(total * k1 / (k1 + k2))), lower), upper)
    in_sub = np.zeros(len(node_w), dtype=bool)
    in_sub[subset] = True
    taken = np.zeros(len(node_w), dtype=bool)
    queue, left, w, pos, head = [], [], 0, 0, 0
    while w < target:
        if head >= len(queue):
            while pos < len(subset) and taken[subset[pos]]:
                pos += 1
            if pos >= len(subset):
                break
            queue.append(int(subset[pos]))
            taken[subset[pos]] = True
        u = queue[head]
        head += 1
        if w + node_w[u] > upper:
            continue
        left.append(u)
        w += int(node_w[u])
        for v in indices[indptr[u]:indptr[u + 1]]:
            if in_sub[v] and not taken[v]:
                taken[v] = True
                queue.append(int(v))
    mask = np.zeros(len(node_w), dtype=bool)
    mask[np.asarray(left, dtype=np.int64)] = True
    return np.asarray(sorted(left), dtype=np.int64), subset[~mask[subset]]


def initial_partition(indptr, indices, node_w, num_blocks, cap):
    """partition.py:239-252."""
    a = np.full(len(node_w), -1, dtype=np.int64)

    def rec(subset, first, k):
        if k == 1 or len(subset) == 0:
            a[subset] = first
            return
        k1 = (k + 1) // 2
        left, right = grow_bisection(indptr, indices, node_w, subset, k1, k - k1, cap)
        rec(left, first, k1)
        rec(right, first + k1, k - k1)

    rec(np.arange(len(node_w), dtype=np.int64), 0, num_blocks)
    return a


def rebalance(indptr, indices, weights, a, bw, node_w, cap, use_w):
    """partition.py:255-285 (mutates a, bw)."""
    nb = len(bw)
    guard = 0
    while True:
        over = np.flatnonzero(bw > cap)
        if len(over) == 0 or guard > len(a) * 4:
            break
        guard += 1
        b = int(over[0])
        moved = False
        for u in np.flatnonzero(a == b):
            if bw[b] <= cap:
                break
            conn = np.zeros(nb, dtype=np.int64)
            for j in range(indptr[u], indptr[u + 1]):
                conn[a[indices[j]]] += weights[j] if use_w else 1
            conn[b] = -1
            cand = np.flatnonzero(bw + node_w[u] <= cap)
            cand = cand[cand != b]
            if len(cand) == 0:
                continue
            best = cand[np.lexsort((cand, -conn[cand]))][0]
            a[u] = best
            bw[b] -= node_w[u]
            bw[best] += node_w[u]
            moved = True
        if not moved:
            break

"""Oracle loop executors (test infrastructure only -- see oracle/__init__.py).

Inputs are plain arrays: ``table`` (n, arity) int64 mapping, ``ind``
(npts, ic) indirectly read values or None, ``dirv`` (n, dc) direct values,
``inc`` (npts, oc) initial increment-array values.  Each function returns a
new ``inc`` array.
"""

import numpy as np


def element_increments(op: str, ind_rows, dirv, unit: bool, dtype) -> np.ndarray:
    """(batch, arity, comps) increments of the registered loops.

    Restates bench_kernels.py:170-181 (flux, flux-noread), 196-201
    (scatter8) and 226-238 (face-flux, heavy) expression for expression.
    ``ind_rows`` is the gathered (batch, arity, comps) read.
    """
    dt = np.dtype(dtype)
    nb = dirv.shape[0]
    if op in ("flux", "flux-noread"):
        if unit:
            return np.ones((nb, 2, 4), dtype=dt)
        if op == "flux-noread":
            lft = np.repeat(dirv[:, 0:1], 4, axis=1)
            rgt = np.repeat(dirv[:, 1:2], 4, axis=1)
        else:
            lft = (ind_rows[:, 1, :] - ind_rows[:, 0, :]) * dirv[:, 0:1]
            rgt = -lft
        return np.stack([lft, rgt], axis=1)
    if op == "scatter8":
        if unit:
            return np.ones((nb, 8, 3), dtype=dt)
        s = dirv
        v = np.stack([s[:, 0] + s[:, 1], s[:, 1] * s[:, 2], s[:, 3] - s[:, 0]], axis=1)
        return np.repeat(v[:, None, :], 8, axis=1)
    if op in ("face-flux", "face-flux-heavy"):
        if unit:
            return np.ones((nb, 2, 5), dtype=dt)
        sl, sr = ind_rows[:, 0, :], ind_rows[:, 1, :]
        phi = (sr[:, :5] - sl[:, :5]) * dirv[:, 0:1]
        if op == "face-flux-heavy":
            scale = np.sqrt(np.abs(sl[:, 5:6]) + 1) + np.sqrt(np.abs(sr[:, 6:7]) + 2)
            phi = (phi * scale / np.sqrt(dirv[:, 1:2] * dirv[:, 1:2] + 1)).astype(dt)
        return np.stack([phi, -phi], axis=1)
    raise ValueError(f"unknown op {op!r}")


def _gather(table, ind, lo, hi):
    return None if ind is None else ind[table[lo:hi]]


def serial_loop(op, table, ind, dirv, inc, unit=False):
    """execute_serial (simulator.py:215-242): one gather, one evaluation,
    ordered np.add.at in (element, slot) order."""
    out = np.array(inc, copy=True)
    n = table.shape[0]
    if n:
        d = element_increments(op, _gather(table, ind, 0, n), dirv, unit, out.dtype)
        np.add.at(out, table.ravel(), d.reshape(-1, out.shape[1]))
    return out


def global_loop(op, table, ind, dirv, inc, colour_offsets, unit=False):
    """execute_global (simulator.py:382-418): colour ranges in order."""
    out = np.array(inc, copy=True)
    for c in range(len(colour_offsets) - 1):
        lo, hi = int(colour_offsets[c]), int(colour_offsets[c + 1])
        if hi <= lo:
            continue
        d = element_increments(op, _gather(table, ind, lo, hi), dirv[lo:hi], unit, out.dtype)
        np.add.at(out, table[lo:hi].ravel(), d.reshape(-1, out.shape[1]))
    return out


def hier_loop(op, table, ind, dirv, inc, block_offsets, block_colours, thread_colours, staged, written, unit=False):
    """execute_hierarchical (simulator.py:613-654): blocks in (colour, id)
    order; shared region zeroed; thread colours applied in order; then
    out[written] += shared[slot]."""
    out = np.array(inc, copy=True)
    nb = len(block_offsets) - 1
    s_ptr, s_ids = staged
    w_ptr, w_ids = written
    for b in np.lexsort((np.arange(nb), block_colours)):
        lo, hi = int(block_offsets[b]), int(block_offsets[b + 1])
        d = element_increments(op, _gather(table, ind, lo, hi), dirv[lo:hi], unit, out.dtype)
        lst = s_ids[s_ptr[b]:s_ptr[b + 1]]
        shared = np.zeros((lst.size, out.shape[1]), dtype=out.dtype)
        local = np.searchsorted(lst, table[lo:hi])
        tc = thread_colours[lo:hi]
        for c in range(int(tc.max()) + 1 if tc.size else 0):
            mask = tc == c
            if mask.any():
                np.add.at(shared, local[mask].ravel(), d[mask].reshape(-1, out.shape[1]))
        wr = w_ids[w_ptr[b]:w_ptr[b + 1]]
        if wr.size:
            out[wr] += shared[np.searchsorted(lst, wr)]
    return out


def useful_bytes(n_elems, arity, arrays) -> int:
    """Paper formula (simulator.py:315-328): arrays = [(rows, comps, itemsize, incremented)]."""
    total = sum((2 if inc else 1) * rows * comps * isz for rows, comps, isz, inc in arrays)
    return total + n_elems * arity * 4

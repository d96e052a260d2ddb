"""Device plan builder: the reference planner's steps, run on the GPU.

Each step cites the reference function whose result it reproduces
bit for bit (pkg/src/meshplan/plan.py, reorder.py, colouring.py):

=======================  ==========================================  ==================
step                      reference                                   where it runs
=======================  ==========================================  ==================
point graph               reorder.mesh_to_graph (63-79)               GPU (sort/unique)
GPS levels + root         reorder.gps_renumber (95-141)               GPU BFS (native)
element lex sort          reorder.lex_sort_elements (161-171)         GPU stable sorts
chunk / structured        partition.chunk_partition, structured       host arithmetic
split oversized           plan._split_oversized (451-464)             host (nb-sized)
per-block written lists   plan._colour_blocks_ns (241-257)            GPU, CTA per block
block colouring           greedy_colour_csr least-loaded              GPU (sorts + one warp)
thread colouring + sort   plan._thread_colours_for_block (260-284)    GPU, warp per block
staged / written CSR      plan._per_block_point_lists (582-603)       GPU, CTA per block
shared slots              HierarchicalPlan.staged_slots (168-182)     GPU (materialised)
element colouring         plan._colour_elements (232-238)             native host C++
dataflow DAG + order      (new: the dataflow schedule)                GPU
=======================  ==========================================  ==================

Device tensors that the executors need stay resident in a ``DevicePlan``.
"""

from dataclasses import dataclass

import ctypes
import os

import numpy as np
import torch

from . import _native
from .errors import CapacityError, KernelSpecError, MeshValidationError
from .mesh import Mapping, Mesh

DEV = "cuda"


def _dev() -> torch.device:
    _native.require_cuda()
    return torch.device(DEV)


def upload(a: np.ndarray, dev) -> torch.Tensor:
    """Host array -> device tensor; read-only arrays (mesh tables are frozen)
    are copied from without torch's non-writable-array warning."""
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.as_tensor(a, device=dev)


def _sp():
    return _native.stream_ptr()


def single_mapping(mesh: Mesh, kernel) -> Mapping | None:
    """The one mapping a device-executable loop may use (None: no indirection)."""
    names = kernel.mapping_names()
    if not names:
        return None
    if len(names) > 1:
        raise KernelSpecError(
            f"kernel {kernel.name!r} uses {len(names)} mappings; the device engine runs single-mapping loops"
        )
    return mesh.mappings[names[0]]


def slot_mask(kernel, mesh, args) -> int:
    mask = 0
    for a in args:
        for s in kernel.arg_slots(mesh, a):
            mask |= 1 << int(s)
    return mask


def stage_reads(kernel, mesh, staging: str, smask: int) -> bool:
    """Whether the executors stage the indirect read rows in shared memory:
    always under all-indirect staging, and under increment-only staging when
    every read slot is also a staged (incremented) slot of the same mapping:
    the read rows are then in the block's staged list anyway, and taking them
    from shared memory instead of global (simulator.py:605-610) changes no
    value -- the plan is untouched, only the executor's data movement."""
    if staging == "all-indirect":
        return True
    reads = list(kernel.indirect_read_args)
    if not reads or smask == 0:
        return False
    return slot_mask(kernel, mesh, reads) & ~smask == 0


# ---------------------------------------------------------------------------------
# reorderings
# ---------------------------------------------------------------------------------


def point_graph(map_d: torch.Tensor, npts: int):
    """Union of per-element cliques (reorder.py:63-79) as a device CSR."""
    rows = map_d.long()
    ar = rows.shape[1]
    us, vs = [], []
    for a in range(ar):
        for b in range(a + 1, ar):
            u, v = rows[:, a], rows[:, b]
            keep = u != v
            us.append(u[keep])
            vs.append(v[keep])
    if us:
        u = torch.cat(us)
        v = torch.cat(vs)
        keys = torch.unique(torch.cat([u * npts + v, v * npts + u]))
    else:
        keys = torch.empty(0, dtype=torch.long, device=map_d.device)
    src = torch.div(keys, npts, rounding_mode="floor")
    dst = keys - src * npts
    indptr = torch.zeros(npts + 1, dtype=torch.long, device=map_d.device)
    if keys.numel():
        indptr[1:] = torch.cumsum(torch.bincount(src, minlength=npts), 0)
    return indptr, dst.to(torch.int32)


def bfs(indptr, indices, start: int, levels: torch.Tensor) -> tuple:
    n = indptr.numel() - 1
    ecc = np.zeros(1, dtype=np.int32)
    vis = np.zeros(1, dtype=np.int32)
    _native.call("mp_bfs_levels", n, _native.ptr(indptr), _native.ptr(indices), int(start), _native.ptr(levels),
                 ecc.ctypes.data, vis.ctypes.data, _sp())
    return int(ecc[0]), int(vis[0])


def gps_forward(map_d: torch.Tensor, npts: int) -> torch.Tensor:
    """Forward point permutation of gps_renumber (reorder.py:115-141)."""
    indptr, indices = point_graph(map_d, npts)
    return gps_forward_graph(indptr, indices, npts)


def gps_forward_graph(indptr: torch.Tensor, indices: torch.Tensor, npts: int) -> torch.Tensor:
    """gps_renumber (reorder.py:115-141) on a device CSR point graph (int64
    indptr, int32 indices): components by lowest index, pseudo-peripheral
    root, order by (component, level, degree, id)."""
    dev = indptr.device
    deg = indptr[1:] - indptr[:-1]
    comp = torch.arange(npts, dtype=torch.long, device=dev)  # component min id (singletons: self)
    level = torch.zeros(npts, dtype=torch.long, device=dev)
    assigned = deg == 0
    lv = torch.empty(npts, dtype=torch.int32, device=dev)
    ids = torch.arange(npts, dtype=torch.long, device=dev)
    big = torch.iinfo(torch.long).max
    while True:
        free = torch.nonzero(~assigned)
        if free.numel() == 0:
            break
        start = int(free[0, 0])
        bfs(indptr, indices, start, lv)
        in_comp = lv >= 0
        cmin = start  # BFS from the lowest unassigned index: it is the component minimum
        # pseudo-peripheral root (reorder.py:95-112): min (deg, id) start, then
        # farthest-level min (deg, id) while the eccentricity grows
        key = torch.where(in_comp, deg * npts + ids, torch.full_like(ids, big))
        u = int(torch.argmin(key))
        ecc, _ = bfs(indptr, indices, u, lv)
        best = lv.clone()
        while True:
            last = best == ecc
            key = torch.where(last, deg * npts + ids, torch.full_like(ids, big))
            v = int(torch.argmin(key))
            ecc_v, _ = bfs(indptr, indices, v, lv)
            if ecc_v > ecc:
                u, ecc, best = v, ecc_v, lv.clone()
            else:
                break
        comp[in_comp] = cmin
        level[in_comp] = best[in_comp].long()
        assigned |= in_comp
    # order by (component min, level, degree, id): stable LSD passes
    order = ids
    for k in (deg, level, comp):
        _, idx = torch.sort(k[order], stable=True)
        order = order[idx]
    fwd = torch.empty(npts, dtype=torch.long, device=dev)
    fwd[order] = ids
    return fwd


def lex_order(map_d: torch.Tensor, point_fwd: torch.Tensor, npts: int) -> torch.Tensor:
    """Element order of lex_sort_elements (reorder.py:161-171): stable lexsort of
    the sorted renumbered point tuples."""
    keys, _ = torch.sort(point_fwd[map_d.long()], dim=1)
    n, ar = keys.shape
    order = torch.arange(n, dtype=torch.long, device=map_d.device)
    col = ar - 1
    while col >= 0:  # pack two columns per stable pass (npts < 2**31)
        if col >= 1:
            k = keys[:, col - 1] * npts + keys[:, col]
            col -= 2
        else:
            k = keys[:, col]
            col -= 1
        _, idx = torch.sort(k[order], stable=True)
        order = order[idx]
    return order


# ---------------------------------------------------------------------------------
# block-level products
# ---------------------------------------------------------------------------------


def block_points(block_offsets_d, map_d, mask: int, max_block: int):
    """Ascending unique points per block through the masked slots: int32 CSR."""
    nb = block_offsets_d.numel() - 1
    n, ar = map_d.shape
    counts = torch.empty(max(nb, 1), dtype=torch.int32, device=map_d.device)
    off = torch.zeros(nb + 1, dtype=torch.int32, device=map_d.device)
    if nb == 0 or mask == 0:
        return off, torch.empty(0, dtype=torch.int32, device=map_d.device)
    args = (nb, _native.ptr(block_offsets_d), _native.ptr(map_d), n, ar, _native.MP_AOS, mask, int(max_block))
    _native.call("mp_plan_block_points", *args, _native.ptr(counts), None, None, _sp())
    off[1:] = torch.cumsum(counts[:nb], 0, dtype=torch.int32)
    total = int(off[-1])
    ids = torch.empty(max(total, 1), dtype=torch.int32, device=map_d.device)
    _native.call("mp_plan_block_points", *args, _native.ptr(counts), _native.ptr(off), _native.ptr(ids), _sp())
    return off, ids[:total]


def thread_colours(block_offsets_d, map_d, written_mask: int, max_block: int):
    """Per-block smallest-last/first-fit colours, counts and the stable colour sort."""
    nb = block_offsets_d.numel() - 1
    n, ar = map_d.shape
    dev = map_d.device
    cols = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    counts = torch.zeros(max(nb, 1), dtype=torch.int32, device=dev)
    order = torch.arange(max(n, 1), dtype=torch.int32, device=dev)
    if nb and n:
        _native.call("mp_plan_thread_colours", nb, _native.ptr(block_offsets_d), _native.ptr(map_d), n, ar,
                     _native.MP_AOS, written_mask, int(max_block), _native.ptr(cols), _native.ptr(counts),
                     _native.ptr(order), _sp())
    return cols[:n], counts[:nb], order[:n]


def local_slots(block_offsets_d, map_d, mask, st_off, st_ids, wr_off, wr_ids):
    nb = block_offsets_d.numel() - 1
    n, ar = map_d.shape
    dev = map_d.device
    ls = torch.full((max(n * ar, 1),), -1, dtype=torch.int16, device=dev)
    ws = torch.full((max(wr_ids.numel(), 1),), -1, dtype=torch.int16, device=dev)
    if nb:
        _native.call("mp_plan_local_slots", nb, _native.ptr(block_offsets_d), _native.ptr(map_d), n, ar,
                     _native.MP_AOS, mask, _native.ptr(st_off), _native.ptr(st_ids), _native.ptr(ls),
                     _native.ptr(wr_off), _native.ptr(wr_ids), _native.ptr(ws), _sp())
    return ls, ws


def colour_blocks_device(wr_off: torch.Tensor, wr_ids: torch.Tensor, least_loaded: bool = True):
    """Greedy colouring of the blocks over their written points
    (plan._colour_blocks_ns, plan.py:241-257: greedy_colour_csr with blocks as
    items, then relabel by load) on the GPU (``mp_plan_block_colours``).
    Returns the device int64 colours (relabelled by descending load when
    least-loaded, ties by old id: colouring._relabel_by_load, colouring.py:68-74),
    the colour count and the per-colour counts (host int64)."""
    nb = wr_off.numel() - 1
    dev = wr_off.device
    if nb <= 0:
        e = np.empty(0, dtype=np.int64)
        return torch.empty(0, dtype=torch.int64, device=dev), 0, e
    raw = torch.empty(nb, dtype=torch.int32, device=dev)
    ncol = np.zeros(1, dtype=np.int32)
    _native.call("mp_plan_block_colours", nb, _native.ptr(wr_off), _native.ptr(wr_ids), int(bool(least_loaded)),
                 _native.ptr(raw), ncol.ctypes.data, _sp())
    num = int(ncol[0])
    raw = raw.long()
    counts = torch.bincount(raw, minlength=num).cpu().numpy()
    if not least_loaded:
        return raw, num, counts
    rank = np.lexsort((np.arange(num), -counts))
    new_id = np.empty(num, dtype=np.int64)
    new_id[rank] = np.arange(num, dtype=np.int64)
    return torch.as_tensor(new_id, device=dev)[raw], num, counts[rank]


DATAFLOW_LAG = int(__import__("os").environ.get("MESHPLAN_DATAFLOW_LAG", "4096"))


def block_dag(wr_off, wr_ids, npts: int, block_colours_d, ncol: int, lag: int = DATAFLOW_LAG):
    """Predecessor lists (lower-colour blocks sharing a written point) and a
    topological block order: key(b) = max(b, max over preds key(p) + lag),
    blocks sorted by (key, id).  ``lag`` keeps a dependent block about one
    wave of resident CTAs behind its predecessors (so it rarely waits) while
    its shared rows are still in L2."""
    nb = wr_off.numel() - 1
    dev = wr_off.device
    pred_off = torch.zeros(nb + 1, dtype=torch.int32, device=dev)
    order = torch.arange(max(nb, 1), dtype=torch.int32, device=dev)
    if nb == 0:
        return pred_off, torch.zeros(1, dtype=torch.int32, device=dev), order[:0]
    cap = 16 * nb + 1024
    while True:
        preds = torch.zeros(cap, dtype=torch.int32, device=dev)
        npred = np.zeros(1, dtype=np.int64)
        _native.call("mp_plan_block_dag", nb, _native.ptr(wr_off), _native.ptr(wr_ids), int(npts),
                     _native.ptr(block_colours_d), int(ncol), int(lag), _native.ptr(pred_off), _native.ptr(preds),
                     cap, npred.ctypes.data, _native.ptr(order), _sp())
        if int(npred[0]) <= cap:
            return pred_off, preds[: max(int(npred[0]), 1)], order[:nb]
        cap = int(npred[0])


def split_oversized(offsets: np.ndarray, limit: int) -> np.ndarray:
    """plan._split_oversized (451-464): halve any span wider than limit at
    lo + (hi-lo+1)//2, depth first; only oversized spans are touched."""
    sizes = np.diff(offsets)
    if sizes.size == 0 or sizes.max() <= limit:
        return offsets.astype(np.int64)
    out = [int(offsets[0])]
    big = set(np.flatnonzero(sizes > limit).tolist())
    for b in range(sizes.size):
        end = int(offsets[b + 1])
        if b not in big:
            out.append(end)
            continue
        pending = [(out[-1], end)]
        while pending:
            lo, hi = pending.pop(0)
            if hi - lo > limit:
                mid = lo + (hi - lo + 1) // 2
                pending = [(lo, mid), (mid, hi)] + pending
            else:
                out.append(hi)
    return np.asarray(out, dtype=np.int64)


@dataclass
class SubPlan:
    """A block subset of a DevicePlan (DevicePlan.subset): the C struct, the
    number of kept blocks and colour launches, and the arrays it points to."""

    struct: object
    num_blocks: int
    launches: int
    keep: list


@dataclass
class DevicePlan:
    """Device-resident execution structures of one hierarchical plan."""

    map: torch.Tensor               # (n, arity) int32, plan numbering
    block_offsets: torch.Tensor     # int32 [nb+1]
    meta: torch.Tensor              # int32 [nb, 4] {e0, k, s0, ns}
    staged_off: torch.Tensor
    staged_ids: torch.Tensor
    written_off: torch.Tensor
    written_ids: torch.Tensor
    written_slots: torch.Tensor     # int16 (uint16 bits)
    local_slots: torch.Tensor       # uint8 or int16 (uint16 bits) [n*arity]
    thread_colours: torch.Tensor    # uint8 [n]
    colour_counts: torch.Tensor     # int32 [nb]
    block_colours: torch.Tensor     # int32 [nb]
    blocks_by_colour: torch.Tensor  # int32 [nb]
    colour_block_offsets: np.ndarray  # host int32 [ncol+1]
    order: torch.Tensor             # int32 [nb]
    pred_off: torch.Tensor
    preds: torch.Tensor
    flags: torch.Tensor             # int32 [nb] epoch stamps
    tickets: torch.Tensor           # int32 [2]
    block_size: int
    max_staged: int
    stage_reads: bool
    written_is_staged: bool
    npts: int
    pull_off: torch.Tensor | None = None  # int16 (uint16 bits) pull-list offsets
    pull_ref: torch.Tensor | None = None  # int16 local refs e*arity+s
    lag: int = DATAFLOW_LAG
    epoch: int = 0
    tdesc_colour: torch.Tensor | None = None  # int32 [nb][4] per ticket, blocks_by_colour order
    tdesc_order: torch.Tensor | None = None   # int32 [nb][4] per ticket, dataflow order
    elem_meta: torch.Tensor | None = None     # uint8 [n * elem_meta_bytes] slots + colour records
    elem_meta_bytes: int = 0
    tpred_off: torch.Tensor | None = None     # int32 [nb+1] predecessor CSR in ticket order
    tpreds: torch.Tensor | None = None        # int32 block ids
    tpred_pad: torch.Tensor | None = None     # int32 [nb][8] padded predecessor ids
    tblock_colour: torch.Tensor | None = None  # int32 [nb] block of each tdesc_colour entry

    def finish_stream(self) -> None:
        """Streamed-executor structures: ticket descriptors {e0, k | nc << 16,
        s0, ns} in both schedule orders and packed per-element records (arity
        local slots, thread colour byte, first-writer slot mask byte, zero
        padding to a 4-byte multiple)."""
        nb = self.block_offsets.numel() - 1
        dev = self.meta.device
        base = self.meta.clone()
        if nb:
            base[:, 1] |= self.colour_counts.to(torch.int32) << 16
        bbc = self.blocks_by_colour.long()
        self.tdesc_colour = base[bbc].contiguous() if nb else base
        self.tblock_colour = bbc.to(torch.int32).contiguous() if nb else self.blocks_by_colour
        self.tdesc_order = base[self.order.long()].contiguous() if nb else base
        # predecessor lists in ticket order (one indirection less for the sync warp)
        po = self.pred_off.long()
        cnt = (po[1:] - po[:-1])[self.order.long()] if nb else po[:0]
        toff = torch.zeros(nb + 1, dtype=torch.long, device=dev)
        if nb:
            toff[1:] = torch.cumsum(cnt, 0)
        total = int(toff[-1]) if nb else 0
        if total:
            src_start = po[:-1][self.order.long()]
            rel = torch.arange(total, device=dev) - torch.repeat_interleave(toff[:-1], cnt)
            idx = torch.repeat_interleave(src_start, cnt) + rel
            self.tpreds = torch.cat([self.preds.long()[idx].to(torch.int32), torch.zeros(1, dtype=torch.int32, device=dev)])
        else:
            self.tpreds = torch.zeros(1, dtype=torch.int32, device=dev)
        self.tpred_off = toff.to(torch.int32)
        pad = torch.full((max(nb, 1), 8), -1, dtype=torch.int32, device=dev)
        if total:
            slot = torch.arange(total, device=dev) - torch.repeat_interleave(toff[:-1], cnt)
            owner = torch.repeat_interleave(torch.arange(nb, device=dev), cnt)
            keep = slot < 8
            pad[owner[keep], slot[keep]] = self.tpreds[:total][keep]
            pad[cnt > 8, 7] = -2
        self.tpred_pad = pad.reshape(-1).contiguous()
        n = int(self.block_offsets[-1]) if nb else 0
        arity = self.map.shape[1]
        sb = self.local_slots.element_size()
        em = (arity * sb + 2 + 3) & ~3
        rec = torch.zeros(n + 4, em, dtype=torch.uint8, device=dev)
        if n:
            ls = self.local_slots[: n * arity].contiguous()
            rec[:n, : arity * sb] = ls.view(torch.uint8).view(n, arity * sb)
            rec[:n, arity * sb] = self.thread_colours[:n]
            if arity <= 8:
                # first writer of each staged row within its block, in (element,
                # slot) order = thread-colour order: it stores (0 + x) instead of
                # adding into a zeroed row
                slot = (ls.view(torch.int16).long() & 0xFFFF) if sb == 2 else ls.long()
                sizes = (self.block_offsets[1:] - self.block_offsets[:-1]).long()
                blk = torch.repeat_interleave(torch.arange(nb, device=dev), sizes * arity)
                key = blk * (int(self.max_staged) + 2) + slot
                order = torch.sort(key, stable=True).indices
                sk = key[order]
                first_sorted = torch.ones_like(sk, dtype=torch.bool)
                first_sorted[1:] = sk[1:] != sk[:-1]
                first = torch.zeros(n * arity, dtype=torch.bool, device=dev)
                first[order] = first_sorted
                bits = (first.view(n, arity).long() << torch.arange(arity, device=dev)).sum(1)
                rec[:n, arity * sb + 1] = bits.to(torch.uint8)
        self.elem_meta = rec.reshape(-1)
        self.elem_meta_bytes = em

    def struct(self) -> "_native.MpHierPlan":
        p = _native.MpHierPlan()
        p.num_blocks = self.block_offsets.numel() - 1
        p.block_size = int(self.block_size)
        p.stage_reads = int(self.stage_reads)
        p.max_staged = int(self.max_staged)
        p.slot_bytes = self.local_slots.element_size()
        p.written_is_staged = int(self.written_is_staged)
        for name, t in (("meta", self.meta), ("staged_ids", self.staged_ids), ("written_offsets", self.written_off),
                        ("written_ids", self.written_ids), ("written_slots", self.written_slots),
                        ("local_slots", self.local_slots), ("thread_colours", self.thread_colours),
                        ("colour_counts", self.colour_counts), ("blocks_by_colour", self.blocks_by_colour),
                        ("order", self.order), ("pred_offsets", self.pred_off), ("preds", self.preds),
                        ("flags", self.flags), ("tickets", self.tickets)):
            setattr(p, name, t.data_ptr())
        p.num_block_colours = len(self.colour_block_offsets) - 1
        p.colour_block_offsets_host = self.colour_block_offsets.ctypes.data
        if self.pull_off is not None:
            p.pull_off = self.pull_off.data_ptr()
            p.pull_ref = self.pull_ref.data_ptr()
        if self.elem_meta is None:
            self.finish_stream()
        p.tdesc_colour = self.tdesc_colour.data_ptr()
        p.tdesc_order = self.tdesc_order.data_ptr()
        p.elem_meta = self.elem_meta.data_ptr()
        p.elem_meta_bytes = int(self.elem_meta_bytes)
        p.tpred_offsets = self.tpred_off.data_ptr()
        p.tpreds = self.tpreds.data_ptr()
        p.tpred_pad = self.tpred_pad.data_ptr()
        p.tblock_colour = self.tblock_colour.data_ptr()
        return p

    def subset(self, block_mask: torch.Tensor) -> "SubPlan":
        """A view of the plan restricted to the blocks where ``block_mask`` is
        true, for the colour schedules: the same element, staging and pull
        arrays, with each colour's ticket list cut to the kept blocks (in the
        same order).  Running the views of a split of the blocks one after the
        other runs every block once, each colour race-free; a point touched by
        both views gets the first view's increments first."""
        if self.elem_meta is None:
            self.finish_stream()
        dev = self.blocks_by_colour.device
        nb = self.block_offsets.numel() - 1
        offs = np.asarray(self.colour_block_offsets, dtype=np.int64)
        keep = block_mask.to(dev)[self.blocks_by_colour.long()] if nb else torch.zeros(0, dtype=torch.bool, device=dev)
        idx = torch.nonzero(keep).flatten()
        ticket_colour = np.repeat(np.arange(len(offs) - 1), np.diff(offs))
        kept_colour = ticket_colour[idx.cpu().numpy()]
        sub_offs = np.zeros(len(offs), dtype=np.int32)
        sub_offs[1:] = np.cumsum(np.bincount(kept_colour, minlength=len(offs) - 1))
        bbc = self.blocks_by_colour[idx].contiguous()
        tdesc = self.tdesc_colour.reshape(-1, 4)[idx].contiguous() if nb else self.tdesc_colour
        base = self.struct()
        p = _native.MpHierPlan()
        ctypes.pointer(p)[0] = base
        p.num_blocks = int(idx.numel())
        p.blocks_by_colour = bbc.data_ptr()
        p.colour_block_offsets_host = sub_offs.ctypes.data
        p.tdesc_colour = tdesc.data_ptr()
        p.tblock_colour = bbc.data_ptr()
        return SubPlan(p, int(idx.numel()), int(np.count_nonzero(np.diff(sub_offs))), [bbc, tdesc, sub_offs])

    def gather_refs(self):
        """Ref records of the gather-form executor (``mp_plan_gather_refs``),
        built once from the pull lists: (ref offsets [nb+1], records, widest
        block's position count)."""
        cached = self.__dict__.get("_gather")
        if cached is not None:
            return cached
        if self.pull_off is None or self.pull_ref is None:
            raise KernelSpecError("the gather form needs pull lists: every slot staged and written")
        nb = self.block_offsets.numel() - 1
        dev = self.block_offsets.device
        arity = self.map.shape[1]
        counts = torch.zeros(max(nb, 1), dtype=torch.int32, device=dev)
        args = (nb, _native.ptr(self.block_offsets), _native.ptr(self.staged_off), _native.ptr(self.pull_off),
                _native.ptr(self.pull_ref), int(arity))
        _native.call("mp_plan_gather_refs", *args, None, _native.ptr(counts), None, _sp())
        roff = torch.zeros(nb + 1, dtype=torch.int32, device=dev)
        if nb:
            roff[1:] = torch.cumsum(counts[:nb], 0, dtype=torch.int32)
        total = int(roff[-1])
        refs = torch.full((max(total, 1),), -1, dtype=torch.int32, device=dev)
        _native.call("mp_plan_gather_refs", *args, _native.ptr(roff), _native.ptr(counts), _native.ptr(refs), _sp())
        max_refs = int(counts[:nb].max()) if nb else 0
        self.__dict__["_gather"] = (roff, refs, max_refs)
        return self.__dict__["_gather"]

    def reschedule(self, lag: int) -> None:
        """Recompute the dataflow order for another lag (tuning)."""
        ncol = len(self.colour_block_offsets) - 1
        self.pred_off, self.preds, self.order = block_dag(self.written_off, self.written_ids, self.npts,
                                                          self.block_colours, ncol, lag)
        self.lag = lag
        self.elem_meta = None  # ticket descriptors follow the order
        self.__dict__.pop("_struct", None)


def pull_lists(bo: torch.Tensor, ls16: torch.Tensor, arity: int, st_off: torch.Tensor, counts: torch.Tensor,
               max_staged: int):
    """Per block and staged row, the (element*arity + slot) refs writing the
    row in thread-colour order (elements are colour-sorted, so (element, slot)
    order): the pull form of the colour loop (plan.py:508-517 order,
    simulator.py:634-643 semantics).  None when some slot is not staged."""
    dev = bo.device
    nb = bo.numel() - 1
    n_ref = int(bo[-1]) * arity
    slot = ls16[:n_ref].long()
    if nb == 0 or n_ref == 0 or bool((slot < 0).any()):
        return None, None
    sizes = (bo[1:] - bo[:-1]).long()
    ref_block = torch.repeat_interleave(torch.arange(nb, device=dev), sizes * arity)
    width = max_staged + 1
    key = ref_block * width + slot
    order = torch.sort(key, stable=True).indices
    ref = order - bo.long()[ref_block] * arity  # sorted refs stay inside their block
    cnt = torch.bincount(key, minlength=nb * width).view(nb, width)
    excl = torch.cumsum(cnt, 1) - cnt
    j = torch.arange(width, device=dev)
    valid = j[None, :] <= counts.long()[:, None]
    dest = (st_off[:-1].long() + torch.arange(nb, device=dev))[:, None] + j[None, :]
    off = torch.zeros(int(st_off[-1]) + nb + 8, dtype=torch.int16, device=dev)
    off[dest[valid]] = excl[valid].to(torch.int16)
    ref16 = torch.cat([ref.to(torch.int16), torch.zeros(8, dtype=torch.int16, device=dev)])
    return off, ref16


#: executor layout of the staged rows: bank-group placement (mp_plan_row_placement)
ROW_PLACEMENT = os.environ.get("MESHPLAN_ROW_PLACEMENT", "0") == "1"


def place_rows(bo, st_off, st_ids, ls, arity: int, tcol_sorted):
    """Renumber each block's staged rows for conflict-free quarter-warp
    shared-memory access (``mp_plan_row_placement``): the staged id lists are
    permuted within their blocks and the local slots remapped, consistently
    for every executor structure derived from them.  The plan itself (its
    ascending staged lists, HierarchicalPlan.staged) is unchanged; results are
    bit-identical (a slot is a storage position, not an order)."""
    dev = bo.device
    total = st_ids.numel()
    perm = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    tc = tcol_sorted.to(torch.uint8).contiguous()
    _native.call("mp_plan_row_placement", bo.numel() - 1, _native.ptr(bo), _native.ptr(st_off), _native.ptr(ls),
                 int(arity), _native.ptr(tc), _native.ptr(perm), _sp())
    counts = (st_off[1:] - st_off[:-1]).long()
    base = torch.repeat_interleave(st_off[:-1].long(), counts)
    old = base + perm[:total].long()
    new_ids = st_ids[old]
    inv = torch.empty(total, dtype=torch.long, device=dev)
    inv[old] = torch.arange(total, device=dev) - base  # flattened (block, old local) -> new local
    # remap per (element, slot): old local index -> new local index within the element's block
    n_el = int(bo[-1])
    sizes = (bo[1:] - bo[:-1]).long()
    blk_of_ref = torch.repeat_interleave(torch.arange(bo.numel() - 1, device=dev), sizes * arity)
    lsl = ls[: n_el * arity].long() & 0xFFFF
    staged = lsl != 0xFFFF
    idx = st_off[:-1].long()[blk_of_ref] + torch.where(staged, lsl, torch.zeros_like(lsl))
    new_ls = torch.where(staged, inv[idx], lsl)
    out = ls.clone()
    out[: n_el * arity] = new_ls.to(torch.int16)
    return new_ids.to(torch.int32), out


def build_device_hier(map_d, block_offsets_np, block_colours_np, ncol, tcol_sorted_d, tcounts_d, st_off, st_ids,
                      wr_off, wr_ids, stage_mask, stage_reads, npts, block_size) -> DevicePlan:
    """Assemble the executor structures (slots, schedules) from plan arrays."""
    dev = map_d.device
    bo = torch.as_tensor(block_offsets_np.astype(np.int32), device=dev)
    nb = bo.numel() - 1
    ls, ws = local_slots(bo, map_d, stage_mask, st_off, st_ids, wr_off, wr_ids)
    counts = (st_off[1:] - st_off[:-1]) if nb else torch.zeros(0, dtype=torch.int32, device=dev)
    if ROW_PLACEMENT and nb and torch.equal(st_off, wr_off) and torch.equal(st_ids, wr_ids) and \
            int(counts.max()) <= 4096:
        st_ids, ls = place_rows(bo, st_off, st_ids, ls, map_d.shape[1], tcol_sorted_d)
        wr_ids = st_ids
    max_staged = int(counts.max()) if nb else 0
    arity = map_d.shape[1]
    full_mask = stage_mask == (1 << arity) - 1
    p_off, p_ref = pull_lists(bo, ls, arity, st_off, counts, max_staged) if full_mask else (None, None)
    if max_staged <= 256:
        ls = ls.to(torch.uint8)  # slot values < 256 (unused slots 0xFFFF only where not staged)
    # 16 bytes of tail padding: the pipelined producer copies 4-byte aligned windows
    ls = torch.cat([ls, torch.zeros(16 // ls.element_size(), dtype=ls.dtype, device=dev)])
    tcol_sorted_d = torch.cat([tcol_sorted_d.to(torch.uint8), torch.zeros(16, dtype=torch.uint8, device=dev)])
    wsame = bool(torch.equal(st_off, wr_off) and torch.equal(st_ids, wr_ids))
    pad4 = torch.zeros(4, dtype=torch.int32, device=dev)  # 16-B window over-read slack (pipelined producer)
    st_ids = torch.cat([st_ids, pad4])
    wr_ids = st_ids if wsame else torch.cat([wr_ids, pad4])
    meta = torch.stack([bo[:-1], bo[1:] - bo[:-1], st_off[:-1], counts], dim=1).to(torch.int32).contiguous()
    bc = torch.as_tensor(block_colours_np.astype(np.int32), device=dev)
    by_colour = np.lexsort((np.arange(nb), block_colours_np)).astype(np.int32) if nb else np.zeros(0, np.int32)
    cbo = np.zeros(ncol + 1, dtype=np.int32)
    if nb:
        cbo[1:] = np.cumsum(np.bincount(block_colours_np, minlength=ncol))
    pred_off, preds, order = block_dag(wr_off, wr_ids, npts, bc, ncol)
    if tcounts_d.numel() and int(tcounts_d.max()) > 255:
        raise CapacityError("a block needs more than 255 thread colours")
    return DevicePlan(
        map=map_d, block_offsets=bo, meta=meta, staged_off=st_off, staged_ids=st_ids, written_off=wr_off,
        written_ids=wr_ids, written_slots=ws, local_slots=ls, thread_colours=tcol_sorted_d.to(torch.uint8),
        colour_counts=tcounts_d.to(torch.int32), block_colours=bc,
        blocks_by_colour=torch.as_tensor(by_colour, device=dev), colour_block_offsets=cbo, order=order,
        pred_off=pred_off, preds=preds, flags=torch.zeros(max(nb, 1), dtype=torch.int32, device=dev),
        tickets=torch.zeros(2, dtype=torch.int32, device=dev), block_size=int(block_size), max_staged=max_staged,
        stage_reads=bool(stage_reads), written_is_staged=wsame, npts=int(npts), pull_off=p_off, pull_ref=p_ref,
    )


def check_block_widths(offsets: np.ndarray, limit: int) -> None:
    if offsets.size > 1 and int(np.diff(offsets).max()) > limit:
        raise CapacityError("plan contains a block wider than the configured block size")


def to_host_i64(t: torch.Tensor) -> np.ndarray:
    return t.to(torch.int64).cpu().numpy()


def validate_device_limits(mesh: Mesh, m: Mapping | None) -> None:
    for s in mesh.sets.values():
        if s.size >= 2**31 - 1:
            raise MeshValidationError(f"set {s.name!r} too large for int32 device indices")
    if m is not None and m.arity > 32:
        raise KernelSpecError(f"mapping {m.name!r} arity {m.arity} exceeds the device limit of 32")

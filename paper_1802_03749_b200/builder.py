"""The two plan builders, orchestrating the GPU planner steps (``gpuplan``).

Reference flow: plan.py:408-448 (global) and plan.py:467-579 (hierarchical).
The mapping table lives on the device from the first step; renumberings are
composed as device gathers; only the sequential greedy colourings cross to
the host (as compact CSR arrays).  The plan object returned is the
reference-compatible host view (numpy fields, plan-numbered host mesh in
pinned memory) with the device execution structures attached as
``plan._device``.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import gpuplan
from .colouring import ColourAssignment, colour_csr_least_loaded
from .errors import CapacityError, KernelSpecError, MeshValidationError
from .mesh import DataArray, Mapping, Mesh
from .partition import partition_structured_hex
from .permutation import Permutation
from .plan import GlobalPlan, HierarchicalPlan, _layouts, _refs_per_element

PIN_THRESHOLD = 1 << 20  # host arrays above this many bytes go to pinned memory


@dataclass
class GlobalDevicePlan:
    map: torch.Tensor  # (n, arity) int32, colour-sorted element order
    colour_offsets: np.ndarray


def _host_copy(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> numpy array (pinned when large, so e2e H2D is DMA)."""
    if t.numel() * t.element_size() >= PIN_THRESHOLD:
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h.numpy()
    return t.cpu().numpy()


def _compose(fwd: dict, set_name: str, new_fwd: torch.Tensor) -> None:
    """set perm := set perm then new (Permutation.then, permutation.py:64-66)."""
    old = fwd.get(set_name)
    fwd[set_name] = new_fwd if old is None else new_fwd[old]


def _fwd_from_order(order: torch.Tensor) -> torch.Tensor:
    fwd = torch.empty_like(order)
    fwd[order] = torch.arange(order.numel(), dtype=order.dtype, device=order.device)
    return fwd


def _reorder(mesh, kernel, config, m: Mapping, map_d: torch.Tensor, fwd: dict):
    """Apply the configured renumbering (plan.py:287-378).  Returns the
    renumbered map, per-block sizes (or None for chunking) and partition meta."""
    iter_set = kernel.iter_set_name(mesh)
    npts = m.to_set.size
    mode = config.reorder.split(":", 1)[0]
    if mode in ("gps", "partition", "cluster") and not kernel.indirect_args:
        mode = "none"
    sizes, meta = None, {}
    if mode == "gps":
        pf = gpuplan.gps_forward(map_d, npts)
        order = gpuplan.lex_order(map_d, pf, npts)
        map_d = pf[map_d[order].long()].to(torch.int32)
        _compose(fwd, m.to_set.name, pf)
        _compose(fwd, iter_set, _fwd_from_order(order))
    elif mode == "partition":
        from . import kway

        res = kway.partition_for_plan(map_d, npts, config)
        map_d = res.point_fwd[map_d[res.order].long()].to(torch.int32)
        _compose(fwd, m.to_set.name, res.point_fwd)
        _compose(fwd, iter_set, _fwd_from_order(res.order))
        sizes = res.block_sizes
        meta = res.meta
    elif mode == "cluster":  # extension: parallel GPU clustering blocks (see cluster.py)
        from . import cluster, kway

        pf_gps = gpuplan.gps_forward(map_d, npts)
        gorder = gpuplan.lex_order(map_d, pf_gps, npts)
        rank = torch.empty_like(gorder)
        rank[gorder] = torch.arange(gorder.numel(), device=gorder.device)
        order, _, sizes, meta = cluster.cluster_order(map_d, npts, config.block_size, rank)
        assign = torch.empty_like(order)
        assign[order] = torch.repeat_interleave(
            torch.arange(len(sizes), device=order.device), torch.as_tensor(sizes, device=order.device))
        pf = kway.writer_set_forward(map_d, npts, assign)
        map_d = pf[map_d[order].long()].to(torch.int32)
        _compose(fwd, m.to_set.name, pf)
        _compose(fwd, iter_set, _fwd_from_order(order))
    elif mode == "structured" and mesh.meta.get("family", "") == "quad2d":
        # extension (the reference defines handcrafted blocks for hex meshes
        # only, plan.py:355-363): bx x by cell tiles of a generated quad grid,
        # ragged at the far edges; each edge goes with its owner (first) cell
        # as faces do in partition_structured_hex; points then follow the
        # writer-set order (reorder.py:174-203) so a tile's cells are contiguous
        from . import kway

        shape = config.structured_shape()
        dims = tuple(int(v) for v in str(mesh.meta.get("dims", "")).split())
        if len(dims) != 2 or shape[2:] not in ((), (1,)):
            raise MeshValidationError("structured quad2d blocks need a generated quad mesh and bx,by")
        nx, ny = dims
        bx, by = shape[0], shape[1]
        if bx < 1 or by < 1 or npts != nx * ny:
            raise MeshValidationError(f"block shape {shape} does not fit a {nx}x{ny} quad grid")
        owner = map_d[:, 0].long()
        cx, cy = torch.div(owner, ny, rounding_mode="floor"), owner % ny
        tiles_y = -(-ny // by)
        assign = torch.div(cx, bx, rounding_mode="floor") * tiles_y + torch.div(cy, by, rounding_mode="floor")
        order = torch.sort(assign, stable=True).indices
        counts = torch.bincount(assign, minlength=int(assign.max()) + 1 if assign.numel() else 0)
        sizes = counts[counts > 0].cpu().numpy().astype(np.int64)
        dense = torch.cumsum(counts > 0, 0) - 1  # drop empty tiles from the numbering
        pf = kway.writer_set_forward(map_d, npts, dense[assign])
        map_d = pf[map_d[order].long()].to(torch.int32)
        _compose(fwd, m.to_set.name, pf)
        _compose(fwd, iter_set, _fwd_from_order(order))
        meta = {"num_blocks": int(sizes.size), "block_shape": [bx, by], "method": "quad2d cell tiles (extension)"}
    elif mode == "structured":
        shape = config.structured_shape()
        family, dims = mesh.meta.get("family", ""), mesh.meta.get("dims", "")
        if family not in ("hex3d-nodes", "hex3d-faces") or not dims:
            raise MeshValidationError("structured reorder needs a generated hex mesh with family/dims metadata")
        dims = tuple(int(v) for v in str(dims).split())
        part = partition_structured_hex(dims, shape, "cells-nodes" if family == "hex3d-nodes" else "faces-cells")
        if part.assignment.size != map_d.shape[0]:
            raise MeshValidationError("structured partition does not match the iteration set")
        order_np = np.argsort(part.assignment, kind="stable")
        order = torch.as_tensor(order_np, device=map_d.device)
        map_d = map_d[order]
        _compose(fwd, iter_set, _fwd_from_order(order))
        sizes = part.block_sizes()
        meta = {"num_blocks": part.num_blocks, "block_shape": list(shape)}
    elif mode != "none":
        raise MeshValidationError(f"unknown reorder mode {config.reorder!r}")
    return map_d, sizes, meta


def _materialise(mesh: Mesh, kernel, m: Mapping, map_d: torch.Tensor, fwd: dict, layouts: dict):
    """Host plan mesh (all arrays renumbered + laid out) and host set perms."""
    dev = map_d.device
    inv = {name: _fwd_from_order(f) for name, f in fwd.items()}  # inverse of a forward perm
    perms = {}
    for name, s in mesh.sets.items():
        perms[name] = (Permutation.unchecked(fwd[name].cpu().numpy(), inv[name].cpu().numpy()) if name in fwd
                       else Permutation.identity(s.size))
    maps = []
    for mm in mesh.mappings.values():
        if mm is m:
            maps.append(Mapping(mm.name, mm.from_set, mm.to_set, map_d.to(torch.int64).cpu().numpy()))
            continue
        t = torch.as_tensor(mm.table, device=dev)
        if mm.from_set.name in inv:
            t = t[inv[mm.from_set.name]]
        if mm.to_set.name in fwd:
            t = fwd[mm.to_set.name][t]
        maps.append(Mapping(mm.name, mm.from_set, mm.to_set, t.cpu().numpy()))
    arrays = []
    for name, a in mesh.data.items():
        v = torch.as_tensor(np.ascontiguousarray(a.view2d()), device=dev)
        if a.set.name in inv:
            v = v[inv[a.set.name]]
        lay = layouts.get(name, a.layout)
        flat = v.t().contiguous().reshape(-1) if lay == "soa" else v.reshape(-1)
        arrays.append(DataArray(a.name, a.set, a.components, _host_copy(flat), lay))
    return Mesh.build(list(mesh.sets.values()), maps, arrays, mesh.meta), perms


def _iter_identity(fwd, name, n, dev):
    if name not in fwd:
        fwd[name] = torch.arange(n, dtype=torch.long, device=dev)


def build_global(mesh: Mesh, kernel, config, hw) -> GlobalPlan:
    dev = gpuplan._dev()
    m = gpuplan.single_mapping(mesh, kernel)
    if m is None:
        raise KernelSpecError(f"kernel {kernel.name!r} has no indirect argument to plan")
    gpuplan.validate_device_limits(mesh, m)
    iter_set = kernel.iter_set_name(mesh)
    n = mesh.sets[iter_set].size
    fwd: dict = {}
    map_d = gpuplan.upload(m.table, dev).to(torch.int32).reshape(n, m.arity)
    map_d, _, _ = _reorder(mesh, kernel, config, m, map_d, fwd)

    # per-element distinct written points (plan.py:201-229) -> greedy least-loaded
    wslots = sorted({s for a in kernel.increment_args for s in kernel.arg_slots(mesh, a)})
    rows = torch.sort(map_d[:, wslots].long(), dim=1).values if wslots else map_d[:, :0].long()
    if rows.shape[1]:
        keep = torch.ones_like(rows, dtype=torch.bool)
        keep[:, 1:] = rows[:, 1:] != rows[:, :-1]
        indptr = torch.zeros(n + 1, dtype=torch.long, device=dev)
        indptr[1:] = torch.cumsum(keep.sum(1), 0)
        indices = rows[keep]
    else:
        indptr = torch.zeros(n + 1, dtype=torch.long, device=dev)
        indices = rows.reshape(-1)
    colours = colour_csr_least_loaded(indptr.cpu().numpy(), indices.cpu().numpy(), max(m.to_set.size, 1))
    if n:
        order_np = np.argsort(colours.colours, kind="stable").astype(np.int64)
        order = torch.as_tensor(order_np, device=dev)
        map_d = map_d[order]
        _compose(fwd, iter_set, _fwd_from_order(order))
        sorted_c = colours.colours[order_np]
        offsets = np.zeros(colours.num_colours + 1, dtype=np.int64)
        offsets[1:] = np.cumsum(np.bincount(sorted_c, minlength=colours.num_colours))
        colours = ColourAssignment(sorted_c, colours.num_colours, colours.counts)
    else:
        offsets = np.zeros(1, dtype=np.int64)
    layouts = _layouts(mesh, kernel, config)
    pmesh, perms = _materialise(mesh, kernel, m, map_d, fwd, layouts)
    plan = GlobalPlan(pmesh, kernel.signature_key(), config, hw, perms, colours, offsets, layouts)
    object.__setattr__(plan, "_device", GlobalDevicePlan(map_d.contiguous(), offsets))
    return plan


class PhaseTimer:
    """Wall time of planner phases (device synchronised at each mark)."""

    def __init__(self):
        import time

        self._now = time.perf_counter
        self.t = self._now()
        self.phases = {}

    def mark(self, name):
        torch.cuda.synchronize()
        now = self._now()
        self.phases[name] = round(self.phases.get(name, 0.0) + now - self.t, 4)
        self.t = now


def build_hier(mesh: Mesh, kernel, config, hw) -> HierarchicalPlan:
    dev = gpuplan._dev()
    tm = PhaseTimer()
    m = gpuplan.single_mapping(mesh, kernel)
    if m is None:
        raise KernelSpecError(f"kernel {kernel.name!r} has no indirect argument to plan")
    gpuplan.validate_device_limits(mesh, m)
    iter_set = kernel.iter_set_name(mesh)
    n = mesh.sets[iter_set].size
    S = config.block_size
    fwd: dict = {}
    map_d = gpuplan.upload(m.table, dev).to(torch.int32).reshape(n, m.arity)
    tm.mark("upload")
    map_d, sizes, meta = _reorder(mesh, kernel, config, m, map_d, fwd)
    tm.mark("reorder")

    if sizes is None:  # chunk_partition (partition.py:165-170)
        offsets = np.append(np.arange(0, n, S, dtype=np.int64), n) if n else np.zeros(1, dtype=np.int64)
    else:
        offsets = np.concatenate(([0], np.cumsum(sizes))).astype(np.int64)
        if offsets[-1] != n:
            raise MeshValidationError("partition does not cover the iteration set")
    offsets = gpuplan.split_oversized(offsets, S)
    nb = offsets.size - 1
    max_block = int(np.diff(offsets).max()) if nb else 0
    bo_d = torch.as_tensor(offsets.astype(np.int32), device=dev)

    inc_args = kernel.increment_args
    staged_args = kernel.indirect_args if config.staging == "all-indirect" else inc_args
    wmask = gpuplan.slot_mask(kernel, mesh, inc_args)
    smask = gpuplan.slot_mask(kernel, mesh, staged_args)

    # block colouring over per-block written point sets (plan.py:241-257)
    wr_off, wr_ids = gpuplan.block_points(bo_d, map_d, wmask, max_block)
    tm.mark("written_lists")
    bcol_d, nbcol, bcounts = gpuplan.colour_blocks_device(wr_off, wr_ids)
    block_colours = ColourAssignment(bcol_d.cpu().numpy(), nbcol, bcounts)
    tm.mark("block_colouring")

    # thread colouring + intra-block colour sort (plan.py:508-522)
    cols, tcounts, sorted_order = gpuplan.thread_colours(bo_d, map_d, wmask, max_block)
    so = sorted_order.long()
    tcol_sorted = cols[so]
    if n and not torch.equal(so, torch.arange(n, device=dev)):
        map_d = map_d[so]
        _compose(fwd, iter_set, _fwd_from_order(so))
    tm.mark("thread_colouring")

    # staging lists on the final numbering (the sort is intra-block: written lists are unchanged)
    if smask == wmask:
        st_off, st_ids = wr_off, wr_ids
    else:
        st_off, st_ids = gpuplan.block_points(bo_d, map_d, smask, max_block)
    s_ptr_h = st_off.to(torch.int64).cpu().numpy()
    s_ids_h = st_ids.to(torch.int64).cpu().numpy()
    if smask == wmask:
        w_ptr_h, w_ids_h = s_ptr_h, s_ids_h
    else:
        w_ptr_h = wr_off.to(torch.int64).cpu().numpy()
        w_ids_h = wr_ids.to(torch.int64).cpu().numpy()
    staged = {m.to_set.name: (s_ptr_h, s_ids_h)} if smask else {}
    written = {m.to_set.name: (w_ptr_h, w_ids_h)} if wmask else {}

    per_point = 0
    counted = set()
    for a in staged_args:
        if a.array not in counted:
            counted.add(a.array)
            arr = mesh.data[a.array]
            per_point += arr.components * arr.values.dtype.itemsize
    shared_bytes = (np.diff(s_ptr_h) * per_point).astype(np.int64) if smask else np.zeros(nb, dtype=np.int64)
    limit = hw.shared_bytes_per_sm
    if nb and shared_bytes.max() > limit:
        b = int(shared_bytes.argmax())
        raise CapacityError(f"block {b} needs {int(shared_bytes[b])} shared bytes, over the {limit}-byte limit")

    layouts = _layouts(mesh, kernel, config)
    _iter_identity(fwd, iter_set, n, dev)
    tm.mark("staging_lists")
    pmesh, perms = _materialise(mesh, kernel, m, map_d, fwd, layouts)
    tm.mark("host_plan_mesh")
    plan = HierarchicalPlan(
        pmesh, kernel.signature_key(), config, hw, perms, offsets, block_colours,
        tcol_sorted.to(torch.int64).cpu().numpy(), tcounts.to(torch.int64).cpu().numpy(), staged, written,
        shared_bytes, _refs_per_element(mesh, kernel), meta, layouts,
    )
    dp = gpuplan.build_device_hier(
        map_d.contiguous(), offsets, block_colours.colours, block_colours.num_colours, tcol_sorted, tcounts,
        st_off, st_ids, wr_off, wr_ids, smask, gpuplan.stage_reads(kernel, mesh, config.staging, smask),
        m.to_set.size, max_block,
    )
    tm.mark("device_plan")
    object.__setattr__(plan, "_device", dp)
    object.__setattr__(plan, "_timings", tm.phases)
    return plan

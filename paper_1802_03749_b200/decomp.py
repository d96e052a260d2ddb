"""Owner-compute domain decomposition across GPUs.

The reference is single-process; this is the new
multi-GPU axis.  The to-set (cells) is split into contiguous owner ranges;
every element goes to the owner of its first point.  A rank's local to-set
is its owned points followed by its halo (points its elements touch but
another rank owns), grouped by owner.  One loop step is

  1. import halo of indirectly read data: each owner packs the rows a peer
     imports (mp_halo_pack) and sends them; the importer scatters them into
     its halo rows (mp_halo_unpack, set);
  2. the local hierarchical loop (any plan / schedule) on the local mesh;
  3. export halo increments: the importer packs its halo increment rows and
     sends them to the owner, which folds them in (mp_halo_unpack, add); the
     importer re-zeroes its halo rows (mp_halo_unpack, zero).

Row lists are in the local *plan* numbering (a plan may renumber points,
e.g. GPS), so nothing assumes contiguous halo rows.  Transports:
``TorchDistTransport`` (torch.distributed send/recv: NCCL over NVLink on the
GPU box, gloo on CPU in the tests) and ``ThreadTransport`` (in-process
queues, to run N ranks on one GPU).  Per point, remote contributions are
added after the owner's local loop, so results equal the serial loop exactly
on the generators' 1/1024-grid data and within reassociation tolerance
otherwise.
"""

import ctypes
import queue
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native

TORCH_TO_MP = {torch.float64: _native.MP_F64, torch.float32: _native.MP_F32, torch.int64: _native.MP_I64,
               torch.int32: _native.MP_I32}
SET, ADD, ZERO = 0, 1, 2


@dataclass
class Decomposition:
    rank: int
    world: int
    lo: int                       # owned global point range [lo, hi)
    hi: int
    local_points: np.ndarray      # global ids: owned (ascending) then halo (by owner, then id)
    halo_rows: dict               # peer -> local rows of my halo owned by peer (ascending global id)
    export_rows: dict             # peer -> local rows of my owned points in the peer's halo (same order)
    local_table: np.ndarray       # (local elements, arity) local point ids
    elem_ids: np.ndarray          # global element ids of the local elements

    @property
    def n_owned(self) -> int:
        return self.hi - self.lo

    @property
    def n_local(self) -> int:
        return int(self.local_points.size)

    def renumbered(self, point_fwd: np.ndarray) -> "Decomposition":
        """The same exchange expressed in a plan's point numbering."""
        f = np.asarray(point_fwd)
        return Decomposition(self.rank, self.world, self.lo, self.hi, self.local_points,
                             {p: f[r] for p, r in self.halo_rows.items()},
                             {p: f[r] for p, r in self.export_rows.items()}, self.local_table, self.elem_ids)


def owner_of(points: np.ndarray, bounds: np.ndarray) -> np.ndarray:
    return np.searchsorted(bounds, points, side="right") - 1


def decompose(table: np.ndarray, elem_ids: np.ndarray, bounds, rank: int, world: int, allgather) -> Decomposition:
    """Local numbering and exchange lists for this rank's elements.

    ``table`` holds the rank's elements (global point ids); ``bounds`` the
    owner ranges (world+1 ascending ids); ``allgather(obj)`` returns the list
    of every rank's ``obj`` (a collective over all ranks)."""
    bounds = np.asarray(bounds, dtype=np.int64)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    pts = np.unique(table)
    halo_pts = pts[(pts < lo) | (pts >= hi)]
    own = owner_of(halo_pts, bounds)
    n_owned = hi - lo
    halo_rows = {int(p): n_owned + np.flatnonzero(own == p) for p in np.unique(own).tolist()}
    local_points = np.concatenate([np.arange(lo, hi, dtype=np.int64), halo_pts])
    inside = (table >= lo) & (table < hi)
    local_table = np.where(inside, table - lo, n_owned + np.searchsorted(halo_pts, table)).astype(np.int64)
    everyone = allgather(halo_pts)
    export_rows = {}
    for peer, theirs in enumerate(everyone):
        if peer == rank:
            continue
        theirs = np.asarray(theirs, dtype=np.int64)
        mine = theirs[owner_of(theirs, bounds) == rank]
        if mine.size:
            export_rows[peer] = mine - lo
    return Decomposition(rank, world, lo, hi, local_points, halo_rows, export_rows, local_table,
                         np.asarray(elem_ids, dtype=np.int64))


# ---- device pack / unpack (hand-written kernels; the CPU tests patch these) -----------


def pack_rows(src: torch.Tensor, rows: torch.Tensor, comps: int, out: torch.Tensor) -> None:
    _native.call("mp_halo_pack", TORCH_TO_MP[src.dtype], src.data_ptr(), rows.data_ptr(), rows.numel(), comps,
                 out.data_ptr(), _native.stream_ptr())


def unpack_rows(dst: torch.Tensor, rows: torch.Tensor, comps: int, src, mode: int) -> None:
    _native.call("mp_halo_unpack", TORCH_TO_MP[dst.dtype], dst.data_ptr(), rows.data_ptr(), rows.numel(), comps,
                 None if src is None else src.data_ptr(), mode, _native.stream_ptr())


# ---- transports --------------------------------------------------------------------------


class TorchDistTransport:
    """Point-to-point exchange through torch.distributed (NCCL / gloo)."""

    def exchange(self, send: dict, recv: dict) -> None:
        import torch.distributed as dist

        ops = [dist.P2POp(dist.isend, t, peer) for peer, t in sorted(send.items())]
        ops += [dist.P2POp(dist.irecv, t, peer) for peer, t in sorted(recv.items())]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()


@dataclass
class ThreadHub:
    """Mailboxes connecting the ThreadTransports of one process."""

    boxes: dict = field(default_factory=dict)

    def box(self, src, dst) -> queue.Queue:
        return self.boxes.setdefault((src, dst), queue.Queue())


class ThreadTransport:
    """In-process transport: each simulated rank runs in its own thread."""

    def __init__(self, hub: ThreadHub, rank: int):
        self.hub, self.rank = hub, rank

    def exchange(self, send: dict, recv: dict) -> None:
        copies = {peer: t.clone() for peer, t in send.items()}
        if any(t.is_cuda for t in send.values()):
            torch.cuda.current_stream().synchronize()  # packed and cloned before a peer reads them
        for peer, t in copies.items():
            self.hub.box(self.rank, peer).put(t)
        for peer, t in recv.items():
            t.copy_(self.hub.box(peer, self.rank).get(timeout=120))  # a failed peer raises queue.Empty


class HaloExchange:
    """Halo import of a read array and export of an increment array (AoS rows,
    flat tensors of rows*comps values)."""

    def __init__(self, dec: Decomposition, transport, device):
        self.dec, self.tr, self.dev = dec, transport, torch.device(device)
        as_rows = lambda r: torch.as_tensor(np.asarray(r, dtype=np.int32), device=self.dev)  # noqa: E731
        self.halo = {p: as_rows(r) for p, r in dec.halo_rows.items()}
        self.exports = {p: as_rows(r) for p, r in dec.export_rows.items()}
        self.all_halo = as_rows(np.concatenate(list(dec.halo_rows.values()))) if dec.halo_rows else None
        self._bufs = {}

    def _buf(self, key, n, dtype):
        b = self._bufs.get(key)
        if b is None or b.numel() != n or b.dtype != dtype:
            b = torch.empty(n, dtype=dtype, device=self.dev)
            self._bufs[key] = b
        return b

    def import_rows(self, arr: torch.Tensor, comps: int) -> None:
        send, recv = {}, {}
        for peer, rows in self.exports.items():
            send[peer] = self._buf(("is", peer, comps), rows.numel() * comps, arr.dtype)
            pack_rows(arr, rows, comps, send[peer])
        for peer, rows in self.halo.items():
            recv[peer] = self._buf(("ir", peer, comps), rows.numel() * comps, arr.dtype)
        self.tr.exchange(send, recv)
        for peer, rows in self.halo.items():
            unpack_rows(arr, rows, comps, recv[peer], SET)

    def export_increments(self, arr: torch.Tensor, comps: int) -> None:
        send, recv = {}, {}
        for peer, rows in self.halo.items():
            send[peer] = self._buf(("es", peer, comps), rows.numel() * comps, arr.dtype)
            pack_rows(arr, rows, comps, send[peer])
        for peer, rows in self.exports.items():
            recv[peer] = self._buf(("er", peer, comps), rows.numel() * comps, arr.dtype)
        self.tr.exchange(send, recv)
        for peer, rows in self.exports.items():
            unpack_rows(arr, rows, comps, recv[peer], ADD)
        if self.all_halo is not None:
            unpack_rows(arr, self.all_halo, comps, None, ZERO)

    def launches_per_step(self) -> int:
        return 2 * (len(self.halo) + len(self.exports)) + (1 if self.all_halo is not None else 0)


# ---- peer-memory exchange (graph-capturable; no NCCL on the data path) ----------------


class PeerHub:
    """Mailbox registry of ranks running as threads of one process, each on its
    own device: a mailbox is published as its raw device pointer.  (Ranks
    sharing one device must be processes -- ``ipc_connector``: threads share
    the process's hardware work queues, where one rank's waiting ``get`` can
    hold up another rank's ``put``.)"""

    def __init__(self):
        self._boxes, self._cv = {}, threading.Condition()

    def connector(self, rank: int):
        def publish(ptr: int, layout: dict, needed) -> dict:
            with self._cv:
                self._boxes[rank] = (ptr, layout)
                self._cv.notify_all()
                if not self._cv.wait_for(lambda: all(p in self._boxes for p in needed), timeout=120):
                    raise TimeoutError(f"rank {rank}: peers {sorted(set(needed) - set(self._boxes))} never published")
                return {p: self._boxes[p] for p in needed}

        publish.ipc = False
        return publish


def ipc_connector(allgather):
    """Mailbox publication across processes: each rank shares the IPC handle
    of its mailbox through ``allgather`` (e.g. torch.distributed
    all_gather_object over the launcher's process group) and maps the
    mailboxes of the peers it writes to (P2P over NVLink between devices)."""
    def publish(ptr: int, layout: dict, needed) -> dict:
        h = (ctypes.c_char * 64)()
        _native.call("mp_ipc_handle", ptr, h)
        everyone = allgather((bytes(h), layout))
        out = {}
        for p in needed:
            handle, lay = everyone[p]
            dptr = ctypes.c_void_p()
            _native.call("mp_ipc_open", (ctypes.c_char * 64).from_buffer_copy(handle), ctypes.byref(dptr))
            out[p] = (dptr.value, lay)
        return out

    publish.ipc = True
    return publish


class PeerExchange:
    """Halo import / export through peer memory (SURVEY 8e step two).

    Every rank owns one mailbox (``mp_mailbox_alloc``): two epoch-parity slots
    per (peer, direction) it receives from, one flag per (peer, direction),
    its put completion counters and its step epoch.  ``import_rows`` puts the
    rows each peer imports straight into that peer's mailbox
    (``mp_halo_put``: P2P stores, then a release of the epoch in the peer's
    flag) and waits for / unpacks its own halo rows (``mp_halo_get``);
    ``export_increments`` does the same for halo increments (added by the
    owner) and re-zeroes the halo rows -- or, with ``fused_export``, only
    releases the epoch (``mp_halo_signal``): the loop's write-back has already
    stored the rows into the owners' slots (``export_slots``).  Nothing waits
    on the host, so a whole step is capturable as a CUDA graph
    (``DistributedLoop.capture``).
    ``publish(ptr, layout, needed)`` exchanges mailboxes (``PeerHub`` for
    threads, ``ipc_connector`` for processes)."""

    def __init__(self, dec: Decomposition, publish, device, dtype: torch.dtype, read_comps: int, inc_comps: int,
                 fused_export: bool = False):
        self.dec, self.dev, self.dtype = dec, torch.device(device), dtype
        self.mp_dtype = TORCH_TO_MP[dtype]
        item = torch.empty(0, dtype=dtype).element_size()
        as_rows = lambda r: torch.as_tensor(np.asarray(r, dtype=np.int32), device=self.dev)  # noqa: E731
        self.halo = {p: as_rows(r) for p, r in dec.halo_rows.items()}
        self.exports = {p: as_rows(r) for p, r in dec.export_rows.items()}
        self.all_halo = as_rows(np.concatenate(list(dec.halo_rows.values()))) if dec.halo_rows else None
        self.rc, self.ic = read_comps, inc_comps
        # layout (bytes): slots [2][rows*comps] per (dir, sender); flags [world][2]; counters [world][2]; epoch
        layout, off = {}, 0
        entries = [(("imp", p), len(r) * read_comps) for p, r in sorted(dec.halo_rows.items())] + \
                  [(("exp", p), len(r) * inc_comps) for p, r in sorted(dec.export_rows.items())]
        for (d, p), n in entries:
            layout[f"{d}:{p}"] = (off, n)
            off += 2 * max(n, 1) * item
            off = (off + 255) & ~255
        layout["flags"] = off
        off += dec.world * 2 * 4
        layout["counters"] = off
        off += dec.world * 2 * 4
        layout["epoch"] = off
        off += 256
        ptr = ctypes.c_void_p()
        _native.call("mp_mailbox_alloc", off, ctypes.byref(ptr))
        self.base, self.layout, self.bytes = ptr.value, layout, off
        needed = sorted(set(dec.export_rows) | set(dec.halo_rows))
        self.peers = publish(self.base, layout, needed)  # every rank takes part (a collective)
        self._ipc = getattr(publish, "ipc", False)
        self._opened = [v[0] for v in self.peers.values()] if self._ipc else []
        # fused export: the loop's write-back stores each halo row's final value
        # into its owner's slot; the exchange only signals (mp_halo_signal)
        self.fused = bool(fused_export)
        self.owners = sorted(dec.halo_rows)
        self.export_slots = []   # per owner index: (slot base address, parity stride in bytes)
        for p in self.owners:
            pbase, play = self.peers[p]
            off, n = play[f"exp:{dec.rank}"]
            self.export_slots.append((pbase + off, max(n, 1) * item))

    def _flag(self, base: int, layout: dict, sender: int, d: int) -> int:
        return base + layout["flags"] + (sender * 2 + d) * 4

    @property
    def epoch_ptr(self) -> int:
        return self.base + self.layout["epoch"]

    def bump(self) -> None:
        _native.call("mp_epoch_bump", self.epoch_ptr, _native.stream_ptr())

    def _put(self, arr, rows, comps, peer, d) -> None:
        pbase, play = self.peers[peer]
        off, n = play[f"{'imp' if d == 0 else 'exp'}:{self.dec.rank}"]
        _native.call("mp_halo_put", self.mp_dtype, arr.data_ptr(), rows.data_ptr(), rows.numel(), comps, pbase + off, n,
                     self._flag(pbase, play, self.dec.rank, d),
                     self.epoch_ptr, self.base + self.layout["counters"] + (peer * 2 + d) * 4, _native.stream_ptr())

    def _get(self, arr, rows, comps, peer, d, mode) -> None:
        off, n = self.layout[f"{'imp' if d == 0 else 'exp'}:{peer}"]
        _native.call("mp_halo_get", self.mp_dtype, arr.data_ptr(), rows.data_ptr(), rows.numel(), comps,
                     self.base + off, n, self._flag(self.base, self.layout, peer, d), self.epoch_ptr, mode,
                     _native.stream_ptr())

    def import_rows(self, arr: torch.Tensor, comps: int) -> None:
        for peer, rows in self.exports.items():
            self._put(arr, rows, comps, peer, 0)
        for peer, rows in self.halo.items():
            self._get(arr, rows, comps, peer, 0, SET)

    def export_increments(self, arr: torch.Tensor, comps: int) -> None:
        for peer, rows in self.halo.items():
            if self.fused:  # rows already stored by the loop's write-back
                pbase, play = self.peers[peer]
                _native.call("mp_halo_signal", self._flag(pbase, play, self.dec.rank, 1), self.epoch_ptr,
                             _native.stream_ptr())
            else:
                self._put(arr, rows, comps, peer, 1)
        for peer, rows in self.exports.items():
            self._get(arr, rows, comps, peer, 1, ADD)
        if self.all_halo is not None:
            unpack_rows(arr, self.all_halo, comps, None, ZERO)

    def launches_per_step(self) -> int:
        return 1 + 2 * (len(self.halo) + len(self.exports)) + (1 if self.all_halo is not None else 0)

    def close(self) -> None:
        """Unmap the peers' mailboxes and free this one (after the last step)."""
        for p in self._opened:
            _native.call("mp_ipc_close", p)
        self._opened = []
        if self.base:
            _native.load().mp_free(ctypes.c_void_p(self.base))
            self.base = 0


def slab_bounds(nx: int, ny: int, world: int):
    """Owner ranges of a quad2d mesh cut into x-slabs (cell = x*ny + y)."""
    xs = np.array([(r * nx) // world for r in range(world + 1)], dtype=np.int64)
    return xs * ny, xs


# ---- a decomposed loop -----------------------------------------------------------------


class DistributedLoop:
    """One rank's share of a decomposed flux-type loop: local plan + halo."""

    def __init__(self, mesh_local, kernel, dec: Decomposition, transport, config, schedule="stream",
                 overlap=None, fused_export=None):
        import paper_1802_03749_b200 as mp

        self.plan = mp.build_hierarchical_plan(mesh_local, kernel, config)
        self.loop = mp.bind(self.plan, kernel, schedule=schedule)
        cells = next(iter(mesh_local.mappings.values())).to_set.name
        self.dec = dec.renumbered(self.plan.set_perms[cells].forward)
        self.read = next((a.array for a in kernel.indirect_read_args), None)
        self.inc = kernel.increment_args[0].array
        self.rc = None if self.read is None else mesh_local.data[self.read].components
        self.ic = mesh_local.data[self.inc].components
        # transport: a mailbox publisher (PeerHub.connector / ipc_connector) selects the
        # peer-memory exchange (device-side, graph-capturable); otherwise host-driven
        # send/recv through the given transport
        self.peer = hasattr(transport, "ipc")
        # fused export (SURVEY 8e step two): the streamed colour executor's
        # write-back stores each halo row's final value straight into its
        # owner's mailbox (P2P); needs the peer exchange and AoS rows
        # (an import round each step orders a sender's slot reuse after the
        # owner's read of it, so the fused export needs an indirectly read array)
        stream_colour = schedule in ("stream", "stream-pull") and self.read is not None
        if fused_export is None:
            fused_export = self.peer and stream_colour
        if fused_export and not (self.peer and stream_colour):
            raise ValueError("fused export needs the peer exchange, a streamed colour schedule and an indirect read")
        if self.peer:
            self.halo = PeerExchange(self.dec, transport, "cuda", self.loop.tensors[self.inc].dtype,
                                     self.rc or 0, self.ic, fused_export=fused_export)
        else:
            self.halo = HaloExchange(self.dec, transport, "cuda")
        self.fused = bool(fused_export)
        if self.fused:
            self.export_dest = self._export_dest()
            # the device-resident export descriptor (csrc ExportDesc): dest, 8 slot
            # bases, 8 parity strides, epoch pointer
            if len(self.halo.export_slots) > 8:
                raise ValueError("fused export supports up to 8 owner peers")
            words = np.zeros(1 + 8 + 8 + 1, dtype=np.int64)
            words[0] = self.export_dest.data_ptr()
            for q, (base, stride) in enumerate(self.halo.export_slots):
                words[1 + q], words[9 + q] = base, stride
            words[17] = self.halo.epoch_ptr
            assert words.nbytes == _native.load().mp_export_desc_bytes()
            self.export_desc = torch.as_tensor(words, device="cuda")
        # core / boundary split: core blocks touch no halo point, so
        # they run while the halo import is in flight; the colour schedules only
        if overlap is None:
            overlap = not schedule.endswith("dataflow") and self.read is not None
        self.core = self.boundary = None
        if overlap:
            core = self.core_blocks()
            self.core = self.plan._device.subset(core)
            self.boundary = self.plan._device.subset(~core)
            self.comm = torch.cuda.Stream()

    def _export_dest(self) -> torch.Tensor:
        """Per staged entry of the local plan: (owner index << 24 | row in the
        owner's export slot) where the entry's block is the last writer (the
        highest block colour) of a halo row, else -1."""
        dp = self.plan._device
        dev = dp.staged_ids.device
        st_off = dp.staged_off.long()
        total = int(st_off[-1])
        ids = dp.staged_ids[:total].long()
        nb = st_off.numel() - 1
        blk = torch.repeat_interleave(torch.arange(nb, device=dev), st_off[1:] - st_off[:-1])
        colour = dp.block_colours.long()[blk]
        n_local = self.dec.n_local
        hpeer = torch.full((n_local,), -1, dtype=torch.long, device=dev)
        hpos = torch.zeros(n_local, dtype=torch.long, device=dev)
        for q, p in enumerate(self.halo.owners):
            rows = torch.as_tensor(np.asarray(self.dec.halo_rows[p], dtype=np.int64), device=dev)
            if q > 255 or rows.numel() >= 1 << 24:
                raise ValueError("fused export: too many owners or halo rows")
            hpeer[rows] = q
            hpos[rows] = torch.arange(rows.numel(), device=dev)
        dest = torch.full((max(total, 1) + 4,), -1, dtype=torch.int32, device=dev)
        halo = hpeer[ids] >= 0
        if bool(halo.any()):
            last = torch.full((n_local,), -1, dtype=torch.long, device=dev)
            last.scatter_reduce_(0, ids[halo], colour[halo], reduce="amax")
            mark = halo & (colour == last[ids])
            dest[:total][mark] = ((hpeer[ids[mark]] << 24) | hpos[ids[mark]]).to(torch.int32)
        return dest

    def _run(self, sub=None) -> None:
        if not self.fused:
            self.loop.run(sub=sub)
            return
        dp = self.plan._device
        _native.call("mp_exec_hier_stream_export", self.loop.loop, (sub.struct if sub is not None else dp.struct_cached()),
                     self.loop.schedule, self.export_desc.data_ptr(), _native.stream_ptr())

    def core_blocks(self) -> torch.Tensor:
        """Per block of the local plan: true when none of its elements
        references a halo point (plan numbering)."""
        dp = self.plan._device
        halo = torch.zeros(self.dec.n_local, dtype=torch.bool, device=dp.map.device)
        if self.halo.all_halo is not None:
            halo[self.halo.all_halo.long()] = True
        touch = halo[dp.map.long()].any(1).to(torch.int32)
        bo = dp.block_offsets.long()
        nb = bo.numel() - 1
        per_block = torch.zeros(nb, dtype=torch.int32, device=touch.device)
        if nb:
            blk = torch.repeat_interleave(torch.arange(nb, device=touch.device), bo[1:] - bo[:-1])
            per_block.index_add_(0, blk, touch)
        return per_block == 0

    def step(self) -> None:
        if self.peer:
            self.halo.bump()  # the step's epoch (device counter: graph replays advance it)
        if self.core is None:
            if self.read is not None:
                self.halo.import_rows(self.loop.tensors[self.read], self.rc)
            self._run()
        else:
            cur = torch.cuda.current_stream()
            self.comm.wait_stream(cur)       # this step's inputs are in place
            self.loop.run(sub=self.core)     # enqueued first: runs while the import is in flight
            with torch.cuda.stream(self.comm):
                self.halo.import_rows(self.loop.tensors[self.read], self.rc)
            cur.wait_stream(self.comm)
            self._run(sub=self.boundary)     # the halo rows' last writers export them (fused)
        self.halo.export_increments(self.loop.tensors[self.inc], self.ic)

    def warmup_step(self) -> None:
        """One real step (collective) whose effect on the increment array --
        local increments and the peers' exports -- is undone afterwards:
        primes kernel attributes and allocations before a capture."""
        inc = self.loop.tensors[self.inc]
        saved = inc.clone()
        self.step()
        torch.cuda.current_stream().synchronize()
        inc.copy_(saved)
        torch.cuda.current_stream().synchronize()

    def capture(self, warmup: bool = True):
        """One step as a CUDA graph (peer-memory exchange only: the NCCL /
        thread transports synchronise on the host).  Collective when
        ``warmup`` (every rank runs ``warmup_step`` together first).
        ``replay()`` runs a step on the current stream -- halo puts and
        waits, core and boundary launches, increment export -- with one
        submission.  Ranks that are threads of one process must capture one
        at a time (capture synchronises the device)."""
        if not self.peer:
            raise RuntimeError("capture needs the peer-memory exchange (PeerHub / ipc_connector transport)")
        if warmup:
            self.warmup_step()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            self.step()
        return g

    def step_host(self, inputs: dict, out) -> None:
        """One end-to-end step with host buffers: H2D of this rank's local
        arrays (pinned), the decomposed step, D2H of the increment array."""
        self.loop.run_host_inputs(inputs)
        self.step()
        inc = self.loop.tensors[self.inc]
        out.copy_(inc.reshape(out.shape), non_blocking=True)

    def owned_result(self) -> np.ndarray:
        """Owned rows of the increment array, in the decomposition's (global) order."""
        pf = self.plan.set_perms[next(iter(self.plan.mesh.mappings.values())).to_set.name].forward
        v = self.loop.tensors[self.inc].reshape(-1, self.ic).cpu().numpy()
        return v[pf[: self.dec.n_owned]]

    def launches_per_step(self) -> int:
        if self.core is not None:
            return self.core.launches + self.boundary.launches + self.halo.launches_per_step()
        return self.loop.launches_per_run() + self.halo.launches_per_step()


def local_flux_mesh(table, elem_ids, dec: Decomposition, q_global_rows, w_rows, res_rows):
    """Local mesh of a rank from its element rows and point rows (AoS f64)."""
    import paper_1802_03749_b200 as mp

    edges, cells = mp.MeshSet("edges", table.shape[0]), mp.MeshSet("cells", dec.n_local)
    data = [mp.DataArray("q", cells, 4, np.ascontiguousarray(q_global_rows).reshape(-1)),
            mp.DataArray("res", cells, 4, np.ascontiguousarray(res_rows).reshape(-1)),
            mp.DataArray("w", edges, 2, np.ascontiguousarray(w_rows).reshape(-1))]
    return mp.Mesh.build([edges, cells], [mp.Mapping("e2c", edges, cells, dec.local_table)], data)


# ---- benchmark rank (bench.py --gpus N under torchrun) -----------------------------------


def bench_rank(args, rank: int, world: int) -> int:
    import json
    import os
    import time

    import torch.distributed as dist

    import paper_1802_03749_b200 as mp
    from .workloads import hashed_grid_values, quad2d_table

    bench = __import__("bench")
    local_rank = int(os.environ.get("LOCAL_RANK", rank))
    # MESHPLAN_RANKS_SHARE_DEVICE=1: every rank on cuda:0 with a gloo process
    # group (rendezvous / timing collectives only; the halo data goes through
    # the IPC-mapped mailboxes) -- the N-rank path exercised on a one-GPU box
    shared = os.environ.get("MESHPLAN_RANKS_SHARE_DEVICE") == "1"
    if shared and getattr(args, "transport", "peer") != "peer":
        raise SystemExit("ranks sharing a device need the peer transport (NCCL refuses duplicate GPUs)")
    if shared:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    family, dims, kname, dtype, staging = bench.CONFIGS[args.config]
    if family != "quad2d" or kname != "flux":
        raise SystemExit("the multi-GPU bench decomposes the quad2d flux configs (C1/C5)")
    nx, ny = dims
    bounds, xs = slab_bounds(nx, ny, world)
    t0 = time.perf_counter()
    table, gids = quad2d_table(nx, ny, int(xs[rank]), int(xs[rank + 1]))

    def allgather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    dec = decompose(table, gids, bounds, rank, world, allgather)
    cid = torch.as_tensor(dec.local_points, device=dev)
    q = hashed_grid_values(cid[:, None] * 4 + torch.arange(4, device=dev), 0, 1).cpu().numpy()
    g = torch.as_tensor(gids, device=dev)
    w = hashed_grid_values(g[:, None] * 2 + torch.arange(2, device=dev), 0, 3).cpu().numpy()
    mesh = local_flux_mesh(table, gids, dec, q, w, np.zeros((dec.n_local, 4)))
    kernel = mp.kernel_for_mesh("flux", mesh)
    cfg = mp.PlanConfig(reorder=args.reorder, layout="aos", block_size=args.block_size)
    sched = "stream" if args.schedule == "best" else args.schedule
    transport = ipc_connector(allgather) if getattr(args, "transport", "peer") == "peer" else TorchDistTransport()
    dl = DistributedLoop(mesh, kernel, dec, transport, cfg, sched)
    t_plan = time.perf_counter() - t0
    # peer exchange: the whole step (epoch bump, halo puts / waits, core and
    # boundary launches, export) is one CUDA graph, one submission per step
    graph = dl.capture() if dl.peer else None
    run_step = graph.replay if graph is not None else dl.step
    sampler = bench.ClockSampler(local_rank)
    sampler.start()
    for _ in range(args.warmup):
        run_step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    # host enqueue cost of a step (what bounds strong scaling once the
    # per-GPU loop is ~0.17 ms at 8 GPUs): submissions without waiting
    t_h = time.perf_counter()
    for _ in range(args.steps):
        run_step()
    enqueue_us = (time.perf_counter() - t_h) / args.steps * 1e6
    torch.cuda.synchronize()
    dist.barrier()
    # a rank's share of the loop's bytes; below twice L2 the steps are timed
    # one by one with L2 flushed in between (as bench.py does on one GPU)
    share = (nx * ny * 4 * 8 * 3 + (nx * (ny - 1) + ny * (nx - 1)) * (2 * 8 + 2 * 4)) / world
    flush = bench.L2Flusher(share < 2 * bench.L2_BYTES)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if flush.buf is None:
        a.record()
        for _ in range(args.steps):
            run_step()
        b.record()
        torch.cuda.synchronize()
        step_ms = a.elapsed_time(b) / args.steps
    else:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for ea, eb in evs:
            flush()
            ea.record()
            run_step()
            eb.record()
        torch.cuda.synchronize()
        step_ms = sum(ea.elapsed_time(eb) for ea, eb in evs) / args.steps
    dist.barrier()
    cdev = torch.device("cpu") if shared else dev  # gloo collectives take host tensors
    ms = torch.tensor([step_ms], device=cdev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    clocks = sampler.stop()
    # end to end: pinned host copies of this rank's arrays -> H2D -> step -> D2H
    host = {}
    for name, tns in dl.loop.tensors.items():
        h = torch.empty(tns.numel(), dtype=tns.dtype, pin_memory=True)
        h.copy_(tns.reshape(-1))
        host[name] = h
    out = torch.empty(dl.loop.tensors[dl.inc].numel(), dtype=dl.loop.tensors[dl.inc].dtype, pin_memory=True)
    h2d = sum(h.numel() * h.element_size() for h in host.values())
    d2h = out.numel() * out.element_size()
    torch.cuda.synchronize()
    dist.barrier()
    a.record()
    n_e2e = max(3, args.steps // 2)
    for _ in range(n_e2e):
        dl.step_host(host, out)
    b.record()
    torch.cuda.synchronize()
    ms_e2e = torch.tensor([a.elapsed_time(b) / n_e2e], device=cdev)
    dist.all_reduce(ms_e2e, op=dist.ReduceOp.MAX)
    io = torch.tensor([h2d, d2h], dtype=torch.float64, device=cdev)
    dist.all_reduce(io)
    n_edges = nx * (ny - 1) + ny * (nx - 1)
    ub_total = nx * ny * 4 * 8 * 3 + n_edges * (2 * 8 + 2 * 4)
    peak, kind = bench.hbm_peak()
    gbps = ub_total / (float(ms) * 1e-3) / 1e9
    if rank == 0:
        line = {
            "metric": bench.METRIC, "value": round(gbps, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(float(ms), 5),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": f"{args.config}: quad2d {nx}x{ny} flux f64 decomposed into {world} x-slabs",
                       "strategy": "hier", "reorder": args.reorder, "schedule": sched,
                       "parallelism": f"owner-compute x{world}, " + (
                           "peer-memory halo exchange (P2P puts into IPC-mapped mailboxes, device-side epoch "
                           "flags), each step one CUDA graph" if dl.peer else "NCCL halo exchange"),
                       "host_enqueue_us_per_step": round(enqueue_us, 2),
                       "ranks_share_device": shared,
                       "useful_bytes_per_step": ub_total,
                       "l2": "inputs larger than L2 (no flush)" if flush.buf is None else "flushed between steps"},
            "roofline": {"bound": "hbm", "achieved": round(gbps / world, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(gbps / world / peak, 4), "traffic": None, "peak_kind": kind,
                         "note": "per-GPU share of the whole-job effective bandwidth"},
            "e2e": {"value": round(ub_total / (float(ms_e2e) * 1e-3) / 1e9, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": int(io[0]), "d2h_bytes_per_step": int(io[1]),
                    "ms_per_step": round(float(ms_e2e), 3),
                    "path": "DistributedLoop.step_host on every rank: pinned local arrays -> H2D -> halo + loop -> D2H"},
            "gpu_launches": int(args.steps * dl.launches_per_step()),
            "clocks": clocks,
            "cpu_baseline": None, "plan_build_s": round(t_plan, 2),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0

"""Executors: run a loop under a plan on the GPU (Seam B of the reference).

``execute_global`` / ``execute_hierarchical`` / ``execute_serial`` keep the
reference signatures and return values (simulator.py:215, 355, 525): they
take the plan's host mesh, copy the loop's arrays to the device, launch the
sm_100a executors through the C ABI, copy the incremented array back and
return ``(result_mesh, MetricsReport)`` in plan numbering.  Like the
reference they *check* plans instead of trusting them -- colour races at both
levels, block widths, shared capacity and staging coverage are verified on
the GPU before any output is produced (once per plan object and kernel).

``DeviceLoop`` is the resident form for time-stepping codes and the
benchmark: arrays stay in HBM and ``run()`` only launches.
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native, gpuplan
from .errors import CapacityError, KernelSpecError, RaceError
from .kernelspec import KernelSpec
from .mesh import DataArray, Mesh
from .plan import GlobalPlan, HierarchicalPlan, MAPPING_ENTRY_BYTES, reuse_factor

#: schedule name -> (native schedule, pipelined persistent kernel?)
SCHEDULES = {
    "colour": (_native.MP_SCHED_COLOUR, False),
    "dataflow": (_native.MP_SCHED_DATAFLOW, False),
    "pipelined": (_native.MP_SCHED_COLOUR, True),
    "pipelined-dataflow": (_native.MP_SCHED_DATAFLOW, True),
    "pipelined-pull": (_native.MP_SCHED_COLOUR | _native.MP_SCHED_PULL, True),
    "pipelined-dataflow-pull": (_native.MP_SCHED_DATAFLOW | _native.MP_SCHED_PULL, True),
    "stream": (_native.MP_SCHED_COLOUR, "stream"),
    "stream-dataflow": (_native.MP_SCHED_DATAFLOW, "stream"),
    "stream-pull": (_native.MP_SCHED_COLOUR | _native.MP_SCHED_PULL, "stream"),
    # gather form (exec_hier_gather.cu): lanes own (element, slot) refs, each
    # row's run summed in thread-colour order by a shuffle chain; no colour loop
    "gather": (_native.MP_SCHED_COLOUR, "gather"),
    # comparison baseline (not bit-exact: atomics reassociate): ignores the colouring
    "atomic": (_native.MP_SCHED_COLOUR, "atomic"),
    # comparison baseline (the paper's temporary-array strategy; bit-identical
    # to execute_serial on the plan's numbering): per-(element, slot) temp
    # increments, then a per-point fold in element order
    "temp-array": (_native.MP_SCHED_COLOUR, "temp-array"),
}
TORCH_DTYPES = {"f64": torch.float64, "f32": torch.float32, "i64": torch.int64, "i32": torch.int32}


# ------------------------------------------------------------------------------
# metrics
# ------------------------------------------------------------------------------


@dataclass
class MetricsReport:
    """Plan-derived and measured metrics of one loop execution.

    Field names follow the reference report (simulator.py:264-312).  The
    reference's cache-line transaction counts and bandwidth proxy are a cost
    model of a P100; here those fields stay ``None`` and the measured
    ``device_ms`` / ``effective_gbps`` (useful bytes / device time, the
    paper's formula) replace them.
    """

    strategy: str
    n_elements: int
    num_launches: int
    block_colours: int
    useful_bytes: int
    temp_array_bytes: int
    atomic_ops: int
    occupancy_estimate: float = 0.0
    blocks_per_sm: int = 0
    reuse_factor: float | None = None
    thread_colours_max: int | None = None
    thread_colours_mean: float | None = None
    sync_count: int = 0
    sync_counts: np.ndarray | None = None
    shared_bytes_max: int = 0
    num_blocks: int = 0
    schedule: str | None = None
    device_ms: float | None = None
    effective_gbps: float | None = None
    read_transactions: int | None = None
    write_transactions: int | None = None
    bandwidth_proxy: float | None = None

    @property
    def total_transactions(self) -> int | None:
        """The reference's modelled transaction total (None: no cost model here)."""
        if self.read_transactions is None or self.write_transactions is None:
            return None
        return self.read_transactions + self.write_transactions

    def to_dict(self, timing: bool = False) -> dict:
        """The report as plain values.  Like the reference's (simulator.py:
        298-312) it is a function of the plan and kernel only, so two
        executions of equal plans give equal dicts; the measured
        ``device_ms`` / ``effective_gbps`` are added with ``timing=True``."""
        out = {}
        for k, v in self.__dict__.items():
            if not timing and k in ("device_ms", "effective_gbps"):
                continue
            if isinstance(v, np.ndarray):
                v = v.tolist()
            elif isinstance(v, np.integer):
                v = int(v)
            elif isinstance(v, np.floating):
                v = float(v)
            out[k] = v
        out["total_transactions"] = self.total_transactions
        return out


def useful_bytes(kernel: KernelSpec, mesh: Mesh) -> int:
    """Paper bandwidth numerator (simulator.py:315-328): every array once,
    incremented arrays twice, plus 4-byte mapping entries."""
    total, seen = 0, set()
    for a in kernel.args:
        if a.array in seen:
            continue
        seen.add(a.array)
        arr = mesh.data[a.array]
        total += (2 if a.mode == "increment" else 1) * arr.set.size * arr.components * arr.values.dtype.itemsize
    for name in kernel.mapping_names():
        m = mesh.mappings[name]
        total += m.from_set.size * m.arity * MAPPING_ENTRY_BYTES
    return total


def consumed_bytes(kernel: KernelSpec, mesh: Mesh, strict: bool = False) -> int:
    """Unique bytes the loop must move, the roofline numerator of SURVEY 8(d):
    like ``useful_bytes`` but an indirectly read array counts only the
    components the element function consumes (face-flux reads 5 of the 28
    ``state`` components, the heavy variant 7; bench_kernels.py:233) -- so a
    kernel that gathers only those cannot show more than 100 %.  Direct and
    incremented arrays count whole (increments read and written once), 4-byte
    map entries.  ``strict`` also trims the direct arrays to the consumed
    components (flux reads ``w[:, 0]`` of 2, face-flux ``facew[:, 0]`` of 4;
    bench_kernels.py:177, 233), the floor for a kernel reading SoA planes."""
    op = (kernel.device_op or "").partition(":")[0]
    if op not in _native.OP_SHAPES:
        raise KernelSpecError(f"kernel {kernel.name!r} has no device functor")
    _, rc, dc, ic = _native.OP_SHAPES[op]
    total, seen = 0, set()
    for a in kernel.args:
        if a.array in seen:
            continue
        seen.add(a.array)
        arr = mesh.data[a.array]
        if a.mode == "increment":
            comps = arr.components
        elif a.indirect:
            comps = min(rc, arr.components)
        else:
            comps = min(dc, arr.components) if strict else arr.components
        total += (2 if a.mode == "increment" else 1) * arr.set.size * comps * arr.values.dtype.itemsize
    for name in kernel.mapping_names():
        m = mesh.mappings[name]
        total += m.from_set.size * m.arity * MAPPING_ENTRY_BYTES
    return total


def _alt_costs(kernel, mesh):
    n = mesh.sets[kernel.iter_set_name(mesh)].size
    tb = ops = 0
    for a in kernel.increment_args:
        arr = mesh.data[a.array]
        k = len(kernel.arg_slots(mesh, a))
        tb += n * k * arr.components * arr.values.dtype.itemsize
        ops += n * k * arr.components
    return tb, ops


@dataclass(frozen=True)
class OccupancyEstimate:
    blocks_per_sm: int
    occupancy: float
    fault: str | None = None


def estimate_occupancy(threads: int, shared_bytes: int, regs: int, hw) -> OccupancyEstimate:
    """Resident blocks/SM and warp-rounded occupancy of a launch shape, with
    the fault message of the first per-block limit it breaks
    (simulator.py:57-103; a report field, not a cost model)."""
    if threads < 1 or regs < 1 or shared_bytes < 0:
        raise ValueError("occupancy inputs must be positive")
    warps = -(-threads // hw.warp_size)
    rpb = warps * -(-regs * hw.warp_size // hw.reg_alloc_granularity) * hw.reg_alloc_granularity
    for bad, msg in ((threads > hw.max_threads_per_block,
                      f"block of {threads} threads exceeds the {hw.max_threads_per_block}-thread limit"),
                     (regs > hw.max_registers_per_thread,
                      f"{regs} registers/thread exceeds the {hw.max_registers_per_thread} limit"),
                     (shared_bytes > hw.shared_bytes_per_sm,
                      f"{shared_bytes} shared bytes exceed the {hw.shared_bytes_per_sm}-byte limit"),
                     (rpb > hw.registers_per_sm, f"{rpb} registers/block exceed the {hw.registers_per_sm}/SM limit")):
        if bad:
            return OccupancyEstimate(0, 0.0, msg)
    blocks = min(hw.max_blocks_per_sm, hw.max_threads_per_sm // threads, hw.max_warps_per_sm // warps,
                 hw.registers_per_sm // rpb)
    if shared_bytes > 0:
        blocks = min(blocks, hw.shared_bytes_per_sm // shared_bytes)
    blocks = max(blocks, 0)
    return OccupancyEstimate(int(blocks), float(blocks * warps * hw.warp_size / hw.max_threads_per_sm))


# ------------------------------------------------------------------------------
# binding a kernel to device arrays
# ------------------------------------------------------------------------------


def _roles(kernel: KernelSpec):
    if kernel.device_op is None:
        raise KernelSpecError(
            f"kernel {kernel.name!r} has no device functor; registered ops are {sorted(_native.OPS)} "
            "(there is no CPU fallback)"
        )
    op, _, variant = kernel.device_op.partition(":")
    if op not in _native.OPS:
        raise KernelSpecError(f"unknown device op {kernel.device_op!r}")
    ind = [a for a in kernel.args if a.indirect and a.mode == "read"]
    dirs = [a for a in kernel.args if not a.indirect and a.mode == "read"]
    incs = [a for a in kernel.args if a.mode == "increment"]
    if len(ind) > 1 or len(dirs) != 1 or len(incs) != 1 or any(a.mode == "write" for a in kernel.args):
        raise KernelSpecError(f"kernel {kernel.name!r}: argument shape does not match device op {op!r}")
    return _native.OPS[op], variant == "unit", (ind[0] if ind else None), dirs[0], incs[0]


@dataclass
class DeviceLoop:
    """A kernel bound to a plan with its arrays resident in HBM (plan numbering)."""

    plan: object
    kernel: KernelSpec
    tensors: dict
    loop: _native.MpLoop
    schedule: int = _native.MP_SCHED_COLOUR
    pipelined: bool | str = False  # True: warp-specialised kernel, "stream": streamed kernel
    launches: int = 0
    _keep: list = field(default_factory=list)
    # dataflow schedules: this loop's own epoch-stamped block flags and ticket
    # counters (the plan stays immutable, so plans run concurrently),
    # the plan struct pointing at them, and the event of this loop's last
    # execution (executions of one loop are chained: they share the flags)
    _df_struct: object = None
    _df_state: tuple = ()
    epoch: int = 0
    _df_event: object = None

    def _dataflow(self) -> bool:
        return (not isinstance(self.plan, GlobalPlan) and self.pipelined not in ("atomic", "temp-array")
                and self.schedule & 3 == _native.MP_SCHED_DATAFLOW)

    def run(self, stream=None, sub=None) -> None:
        """Launch one full execution of the loop (all colours); asynchronous.
        ``sub`` (a DevicePlan.subset view, colour schedules only) runs only
        that view's blocks."""
        sp = _native.stream_ptr(stream)
        dp = self.plan._device
        if self.pipelined == "gather":
            roff, refs, max_refs = dp.gather_refs()
            _native.call("mp_exec_hier_gather", self.loop, (sub.struct if sub is not None else dp.struct_cached()),
                         _native.ptr(roff), _native.ptr(refs), int(max_refs), sp)
            return
        if sub is not None:
            if isinstance(self.plan, GlobalPlan) or self.pipelined in ("atomic", "temp-array") or \
                    self.schedule & 3 == _native.MP_SCHED_DATAFLOW:
                raise KernelSpecError("block subsets run under the colour schedules of a hierarchical plan")
            fn = ("mp_exec_hier_stream" if self.pipelined == "stream" else
                  "mp_exec_hier_pipelined" if self.pipelined else "mp_exec_hier")
            _native.call(fn, self.loop, sub.struct, self.schedule, 1, sp)
            return
        if self.pipelined == "atomic":
            _native.call("mp_exec_atomic", self.loop, sp)
        elif self.pipelined == "temp-array":
            off, refs, temp = self._keep[-3:]
            _native.call("mp_exec_serial", self.loop, off.data_ptr(), refs.data_ptr(), temp.data_ptr(), sp)
        elif isinstance(self.plan, GlobalPlan):
            offs = np.ascontiguousarray(dp.colour_offsets, dtype=np.int64)
            _native.call("mp_exec_global", self.loop, offs.ctypes.data, len(offs) - 1,
                         int(self.plan.config.block_size), sp)
        else:
            fn = ("mp_exec_hier_stream" if self.pipelined == "stream" else
                  "mp_exec_hier_pipelined" if self.pipelined else "mp_exec_hier")
            if not self._dataflow():
                _native.call(fn, self.loop, dp.struct_cached(), self.schedule, 1, sp)
                return
            cur = stream if stream is not None else torch.cuda.current_stream()
            if self._df_event is not None:
                cur.wait_event(self._df_event)  # the previous execution released these flags
            self.epoch = self.epoch % 0xFFFFFFFF + 1  # flags hold the last epoch; never 0
            _native.call(fn, self.loop, self._df_struct, self.schedule, self.epoch, sp)
            self._df_event = torch.cuda.Event()
            self._df_event.record(cur)

    def capture(self):
        """One execution captured as a CUDA graph (colour schedules: the
        launches, with their programmatic-dependent edges, replay with one
        submission).  Returns the ``torch.cuda.CUDAGraph``; ``replay()`` runs
        the loop on the current stream's device.  Dataflow schedules stamp a
        fresh epoch per execution and are not capturable."""
        if self._dataflow():
            raise KernelSpecError("dataflow schedules take a new epoch per execution; capture a colour schedule")
        # warm-up outside the capture (kernel attributes, occupancy queries),
        # with the incremented array restored afterwards: capturing has no
        # effect on the bound arrays
        inc = next(a.array for a in self.kernel.args if a.mode == "increment")
        saved = self.tensors[inc].clone()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.run(side)
            self.tensors[inc].copy_(saved)
        torch.cuda.current_stream().wait_stream(side)
        del saved
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run(torch.cuda.current_stream())
        return g

    def run_host_inputs(self, inputs: dict) -> None:
        """Asynchronous H2D of the given arrays (name -> pinned numpy / torch,
        plan numbering) into the bound device tensors."""
        import warnings

        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)  # read-only numpy views of pinned buffers
            for name, host in inputs.items():
                src = torch.from_numpy(host) if isinstance(host, np.ndarray) else host
                self.tensors[name].copy_(src.reshape(self.tensors[name].shape), non_blocking=True)

    def run_host(self, inputs: dict, out, stream=None) -> None:
        """One end-to-end step with host buffers: H2D of the given arrays
        (name -> pinned numpy / torch, plan numbering), the launch, and D2H of
        the incremented array into ``out``; all on one stream, asynchronous."""
        import warnings

        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)  # read-only numpy views of pinned buffers
            for name, host in inputs.items():
                src = torch.from_numpy(host) if isinstance(host, np.ndarray) else host
                self.tensors[name].copy_(src.reshape(self.tensors[name].shape), non_blocking=True)
        self.run(stream)
        inc = next(a.array for a in self.kernel.args if a.mode == "increment")
        dst = torch.from_numpy(out) if isinstance(out, np.ndarray) else out
        dst.copy_(self.tensors[inc].reshape(dst.shape), non_blocking=True)

    def launches_per_run(self) -> int:
        if self.pipelined in ("atomic", "temp-array"):
            n = 1 if self.plan.mesh.sets[self.kernel.iter_set_name(self.plan.mesh)].size else 0
            return n * (2 if self.pipelined == "temp-array" else 1)
        if isinstance(self.plan, GlobalPlan):
            return int(np.count_nonzero(np.diff(self.plan._device.colour_offsets)))
        if self._dataflow():
            return 1 if self.plan.num_blocks else 0
        return int(np.count_nonzero(np.diff(self.plan._device.colour_block_offsets)))


class HostStream:
    """Loop executions streamed over host buffers: every step copies its
    inputs host -> device, runs the loop and copies the incremented array
    back, like ``DeviceLoop.run_host``, but consecutive steps go to
    ``depth`` CUDA streams with their own device arrays, so one step's
    device -> host copy and the next step's host -> device copy and compute
    overlap (the copy engines work both directions at once).  Pass a
    different ``out`` buffer to steps that may be in flight together."""

    def __init__(self, plan, kernel: KernelSpec, schedule: str = "stream", depth: int = 2):
        self.loops = [bind(plan, kernel, schedule=schedule) for _ in range(depth)]
        self.streams = [torch.cuda.Stream() for _ in range(depth)]
        self.k = 0

    def step(self, inputs: dict, out) -> None:
        """Enqueue one step (asynchronous; ``synchronize`` waits for all)."""
        i = self.k % len(self.loops)
        self.k += 1
        s = self.streams[i]
        with torch.cuda.stream(s):
            self.loops[i].run_host(inputs, out, stream=s)

    def wait_on(self, event) -> None:
        for s in self.streams:
            s.wait_event(event)

    def join(self, stream=None) -> None:
        """Make ``stream`` (default: the current one) wait for every step enqueued so far."""
        cur = stream or torch.cuda.current_stream()
        for s in self.streams:
            cur.wait_stream(s)

    def synchronize(self) -> None:
        for s in self.streams:
            s.synchronize()

    def launches_per_step(self) -> int:
        return self.loops[0].launches_per_run()


def _array_tensor(arr: DataArray, dev) -> torch.Tensor:
    host = torch.from_numpy(np.ascontiguousarray(arr.values))
    return host.to(dev, non_blocking=True)


def bind(plan, kernel: KernelSpec, tensors: dict | None = None, schedule: str = "stream") -> DeviceLoop:
    """Bind ``kernel`` to ``plan``; ``tensors`` (name -> device tensor in plan
    numbering and plan layout) default to uploads of ``plan.mesh``.

    ``schedule`` picks the executor (``SCHEDULES``); the default ``"stream"``
    is the streamed colour-schedule kernel, the fastest on every config.
    Dataflow schedules get their own flags and tickets per bound loop, so any
    number of loops may run one plan at once; executions of one loop are
    ordered after each other on the device."""
    if kernel.signature_key() != plan.kernel_key:
        raise KernelSpecError("plan was built for a different kernel signature")
    mesh = plan.mesh
    kernel.validate_against(mesh)
    op, unit, ind, dr, inc = _roles(kernel)
    ensure_device(plan, kernel)
    dev = torch.device("cuda")
    t = dict(tensors or {})
    for a in (ind, dr, inc):
        if a is not None and a.array not in t:
            t[a.array] = _array_tensor(mesh.data[a.array], dev)
    inc_arr = mesh.data[inc.array]
    dtypes = {mesh.data[a.array].elem_type for a in (ind, dr, inc) if a is not None}
    if len(dtypes) != 1:
        raise KernelSpecError(f"kernel {kernel.name!r}: device ops need one element type, got {sorted(dtypes)}")
    m = mesh.mappings[inc.mapping]
    L = _native.MpLoop()
    L.op, L.unit, L.dtype = op, int(unit), _native.DTYPES[inc_arr.elem_type]
    L.ind_layout = _native.LAYOUTS[inc_arr.layout]
    if ind is not None and mesh.data[ind.array].layout != inc_arr.layout:
        raise KernelSpecError("indirect arrays of one loop must share a layout")
    L.n_elems, L.n_points, L.arity = m.from_set.size, m.to_set.size, m.arity
    L.map_layout = _native.MP_AOS
    L.map = plan._device.map.data_ptr()
    if ind is not None:
        L.ind_read = t[ind.array].data_ptr()
        L.ind_read_comps = mesh.data[ind.array].components
    L.dir_read = t[dr.array].data_ptr()
    L.dir_comps = mesh.data[dr.array].components
    L.inc = t[inc.array].data_ptr()
    L.inc_comps = inc_arr.components
    if schedule not in SCHEDULES:
        raise KernelSpecError(f"unknown schedule {schedule!r}; expected one of {sorted(SCHEDULES)}")
    sched, pipelined = SCHEDULES[schedule]
    keep = []
    if pipelined == "temp-array":
        off, refs = _serial_refs(plan._device.map, sorted(kernel.arg_slots(mesh, inc)), m.to_set.size)
        temp = torch.empty(max(m.from_set.size * m.arity * inc_arr.components, 1),
                           dtype=TORCH_DTYPES[inc_arr.elem_type], device=dev)
        keep = [off, refs, temp]
    loop = DeviceLoop(plan, kernel, t, L, sched, pipelined, _keep=keep)
    if loop._dataflow():
        nb = max(plan.num_blocks, 1)
        flags = torch.zeros(nb, dtype=torch.int32, device=dev)
        tickets = torch.zeros(2, dtype=torch.int32, device=dev)
        base = plan._device.struct_cached()
        st = type(base).from_buffer_copy(base)
        st.flags, st.tickets = flags.data_ptr(), tickets.data_ptr()
        loop._df_struct, loop._df_state = st, (flags, tickets)
    return loop


# ------------------------------------------------------------------------------
# device state + verification (once per plan object and kernel)
# ------------------------------------------------------------------------------


def _struct_cached(self):
    s = getattr(self, "_struct", None)
    if s is None:
        s = self.struct()
        self._struct = s
    return s


gpuplan.DevicePlan.struct_cached = _struct_cached


def ensure_device(plan, kernel: KernelSpec) -> None:
    verified = getattr(plan, "_verified", None)
    if verified is not None and kernel.signature_key() in verified:
        return
    _native.require_cuda()
    if getattr(plan, "_device", None) is None:
        object.__setattr__(plan, "_device", _device_from_host(plan, kernel))
    if isinstance(plan, GlobalPlan):
        _verify_global(plan, kernel)
    else:
        _verify_hier(plan, kernel)
    object.__setattr__(plan, "_verified", (verified or set()) | {kernel.signature_key()})


def _kernel_map(plan, kernel) -> torch.Tensor:
    m = gpuplan.single_mapping(plan.mesh, kernel)
    if m is None:
        raise KernelSpecError(f"kernel {kernel.name!r} has no indirect argument")
    return gpuplan.upload(m.table, "cuda").to(torch.int32).contiguous()


def _device_from_host(plan, kernel):
    """Device structures for a plan that was loaded or edited on the host."""
    from .builder import GlobalDevicePlan

    map_d = _kernel_map(plan, kernel)
    if isinstance(plan, GlobalPlan):
        return GlobalDevicePlan(map_d, np.asarray(plan.colour_offsets, dtype=np.int64))
    mesh = plan.mesh
    m = gpuplan.single_mapping(mesh, kernel)
    dev = map_d.device
    offsets = np.asarray(plan.block_offsets, dtype=np.int64)
    gpuplan.check_block_widths(offsets, plan.config.block_size)
    name = m.to_set.name
    i32 = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int32), device=dev)  # noqa: E731
    empty = (np.zeros(len(offsets), dtype=np.int64), np.zeros(0, dtype=np.int64))
    st = plan.staged.get(name, empty)
    wr = plan.written.get(name, empty)
    staged_args = kernel.indirect_args if plan.config.staging == "all-indirect" else kernel.increment_args
    smask = gpuplan.slot_mask(kernel, mesh, staged_args)
    try:
        return gpuplan.build_device_hier(
            map_d, offsets, np.asarray(plan.block_colours.colours, dtype=np.int64), plan.block_colours.num_colours,
            i32(plan.thread_colours), i32(plan.thread_colour_counts), i32(st[0]), i32(st[1]), i32(wr[0]), i32(wr[1]),
            smask, gpuplan.stage_reads(kernel, mesh, plan.config.staging, smask), m.to_set.size,
            int(np.diff(offsets).max()) if offsets.size > 1 else 0,
        )
    except CapacityError as exc:
        raise CapacityError(f"{exc} on set {name!r}") from None


def _race(n_items, ref_off, refs, groups, span, what, fmt):
    pair = np.full(2, -1, dtype=np.int64)
    _native.call("mp_race_check", int(n_items), _native.ptr(ref_off), _native.ptr(refs), _native.ptr(groups),
                 int(span), pair.ctypes.data, _native.stream_ptr())
    if pair[0] >= 0:
        raise RaceError(fmt(int(pair[0]), int(pair[1])))


def _element_refs(plan, kernel, map_d):
    wslots = sorted({s for a in kernel.increment_args for s in kernel.arg_slots(plan.mesh, a)})
    n = map_d.shape[0]
    refs = map_d[:, wslots].contiguous().reshape(-1)
    off = torch.arange(n + 1, dtype=torch.long, device=map_d.device) * len(wslots)
    return off, refs


def _verify_global(plan: GlobalPlan, kernel) -> None:
    dp = plan._device
    n = dp.map.shape[0]
    offs = np.asarray(plan.colour_offsets, dtype=np.int64)
    colour_of = np.repeat(np.arange(len(offs) - 1, dtype=np.int64), np.diff(offs))
    if colour_of.size != n:
        raise RaceError("global colouring: colour ranges do not cover the iteration set")
    g = torch.as_tensor(colour_of, device="cuda")
    off, refs = _element_refs(plan, kernel, dp.map)
    span = int(plan.mesh.mappings[kernel.increment_args[0].mapping].to_set.size) + 1
    _race(n, off, refs, g, span, "global",
          lambda a, b: f"global colouring: elements {a} and {b} share group {int(colour_of[a])} but write a common point")


def _verify_hier(plan: HierarchicalPlan, kernel) -> None:
    dp = plan._device
    offsets = np.asarray(plan.block_offsets, dtype=np.int64)
    n = dp.map.shape[0]
    nb = offsets.size - 1
    if nb and int(np.diff(offsets).max()) > plan.config.block_size:
        raise CapacityError("plan contains a block wider than the configured block size")
    block_of = np.repeat(np.arange(nb, dtype=np.int64), np.diff(offsets))
    tmax = int(np.asarray(plan.thread_colour_counts).max(initial=0))
    groups = block_of * np.int64(max(tmax, 1) + 1) + np.asarray(plan.thread_colours, dtype=np.int64)
    off, refs = _element_refs(plan, kernel, dp.map)
    m = plan.mesh.mappings[kernel.increment_args[0].mapping]
    span = m.to_set.size + 1
    _race(n, off, refs, torch.as_tensor(groups, device="cuda"), span, "thread",
          lambda a, b: f"thread colouring: elements {a} and {b} share group {int(groups[a])} but write a common point")
    bcol = np.asarray(plan.block_colours.colours, dtype=np.int64)
    for set_name, (indptr, ids) in plan.written.items():
        _race(nb, torch.as_tensor(np.asarray(indptr, dtype=np.int64), device="cuda"),
              torch.as_tensor(np.asarray(ids, dtype=np.int32), device="cuda"), torch.as_tensor(bcol, device="cuda"),
              span, "block",
              lambda a, b, s=set_name: f"block colouring: blocks {a} and {b} share a colour but write a common "
                                       f"point of set {s!r}")
    limit = plan.hw.shared_bytes_per_sm
    if nb and int(plan.shared_bytes.max()) > limit:
        b = int(plan.shared_bytes.argmax())
        raise CapacityError(f"block {b} needs {int(plan.shared_bytes[b])} shared bytes, over the {limit}-byte limit")


# ------------------------------------------------------------------------------
# reference-compatible entry points
# ------------------------------------------------------------------------------


def _report(plan, kernel, loop: DeviceLoop, ms: float | None) -> MetricsReport:
    mesh = plan.mesh
    ub = useful_bytes(kernel, mesh)
    tb, ops = _alt_costs(kernel, mesh)
    n = mesh.sets[kernel.iter_set_name(mesh)].size
    gbps = (ub / (ms * 1e-3) / 1e9) if ms else None
    if isinstance(plan, GlobalPlan):
        est = estimate_occupancy(plan.config.block_size, 0, kernel.regs_per_thread, plan.hw)
        bps, occ = est.blocks_per_sm, est.occupancy
        return MetricsReport("global", n, plan.num_colours, plan.num_colours, ub, tb, ops, occ, bps,
                             num_blocks=int(sum(-(-int(c) // plan.config.block_size) for c in np.diff(plan.colour_offsets))),
                             device_ms=ms, effective_gbps=gbps)
    nb = plan.num_blocks
    sync = plan.thread_colour_counts + 2
    smax = int(plan.shared_bytes.max()) if nb else 0
    est = estimate_occupancy(plan.config.block_size, smax, kernel.regs_per_thread, plan.hw)
    bps, occ = est.blocks_per_sm, est.occupancy
    return MetricsReport(
        "hier", n, loop.launches_per_run(), plan.block_colours.num_colours, ub, tb, ops, occ, bps,
        reuse_factor(plan), int(plan.thread_colour_counts.max()) if nb else 0,
        float(plan.thread_colour_counts.mean()) if nb else 0.0, int(sync.sum()) if nb else 0, sync, smax, nb,
        "gather" if loop.pipelined == "gather" else
        ("stream-" if loop.pipelined == "stream" else "pipelined-" if loop.pipelined else "") + ("dataflow" if loop.schedule & 3 == _native.MP_SCHED_DATAFLOW
                                                    else "colour") + ("-pull" if loop.schedule & 4 else ""),
        ms, gbps,
    )


def _run_and_collect(plan, kernel, schedule="stream"):
    loop = bind(plan, kernel, schedule=schedule)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    loop.run()
    stop.record()
    inc = next(a for a in kernel.args if a.mode == "increment")
    out = loop.tensors[inc.array].cpu().numpy()
    ms = start.elapsed_time(stop)
    arr = plan.mesh.data[inc.array]
    result = plan.mesh.with_data(DataArray(arr.name, arr.set, arr.components, out, arr.layout))
    return result, _report(plan, kernel, loop, ms)


def execute_global(plan: GlobalPlan, kernel: KernelSpec):
    """One launch per colour range; returns (plan-numbered result, report)."""
    if not isinstance(plan, GlobalPlan):
        raise KernelSpecError("execute_global needs a GlobalPlan")
    return _run_and_collect(plan, kernel)


def execute_hierarchical(plan: HierarchicalPlan, kernel: KernelSpec, schedule: str = "stream"):
    """Hierarchical shared-memory execution; ``schedule`` names an executor
    of ``SCHEDULES``: ``"stream"`` (default; one launch per block colour, the
    paper's scheme, persistent streamed kernel), ``"colour"`` (CTA per block),
    the ``"*-dataflow"`` forms (one launch, DAG-ordered blocks) and the
    ``"*-pull"`` forms.  All give bit-identical results."""
    if not isinstance(plan, HierarchicalPlan):
        raise KernelSpecError("execute_hierarchical needs a HierarchicalPlan")
    return _run_and_collect(plan, kernel, schedule)


def _serial_refs(map_d: torch.Tensor, wslots, npts: int):
    """Per point, its (element*arity + slot) references through the written
    slots in element order (np.add.at's order): int32 CSR (offsets, refs)."""
    dev = map_d.device
    n, ar = map_d.shape
    flat = map_d.long().reshape(-1)
    pos = torch.arange(n * ar, dtype=torch.long, device=dev)
    in_w = (pos % max(ar, 1)).unsqueeze(0) == torch.as_tensor(wslots, device=dev).unsqueeze(1) if wslots else None
    sel = in_w.any(0) if in_w is not None else torch.zeros_like(pos, dtype=torch.bool)
    keys, order = torch.sort(flat[sel], stable=True)
    refs = pos[sel][order]
    # temp is indexed by e*arity + s of the op's own slot loop
    off = torch.zeros(npts + 1, dtype=torch.int32, device=dev)
    if keys.numel():
        off[1:] = torch.cumsum(torch.bincount(keys, minlength=npts), 0).to(torch.int32)
    return off, refs.to(torch.int32)


def execute_serial(mesh: Mesh, kernel: KernelSpec) -> Mesh:
    """Element-order semantics of the reference oracle, computed on the GPU:
    temp-array increments + per-point ordered folds (bit-identical to
    np.add.at order for every input)."""
    kernel.validate_against(mesh)
    op, unit, ind, dr, inc = _roles(kernel)
    m = gpuplan.single_mapping(mesh, kernel)
    _native.require_cuda()
    dev = torch.device("cuda")
    n, ar = m.from_set.size, m.arity
    map_d = gpuplan.upload(m.table, dev).to(torch.int32).reshape(n, ar)
    off, refs = _serial_refs(map_d, sorted(kernel.arg_slots(mesh, inc)), m.to_set.size)
    arrays = {}
    for a in (ind, dr, inc):
        if a is not None:
            x = mesh.data[a.array]
            lay = x.layout if a.indirect else "soa"
            v2 = np.ascontiguousarray(x.view2d())
            flat_v = v2.T.ravel() if lay == "soa" else v2.ravel()
            arrays[a.array] = (torch.as_tensor(np.ascontiguousarray(flat_v), device=dev), lay)
    inc_arr = mesh.data[inc.array]
    L = _native.MpLoop()
    L.op, L.unit, L.dtype = op, int(unit), _native.DTYPES[inc_arr.elem_type]
    L.ind_layout = _native.LAYOUTS[arrays[inc.array][1]]
    L.n_elems, L.n_points, L.arity, L.map_layout = n, m.to_set.size, ar, _native.MP_AOS
    L.map = map_d.data_ptr()
    if ind is not None:
        L.ind_read, L.ind_read_comps = arrays[ind.array][0].data_ptr(), mesh.data[ind.array].components
    L.dir_read, L.dir_comps = arrays[dr.array][0].data_ptr(), mesh.data[dr.array].components
    L.inc, L.inc_comps = arrays[inc.array][0].data_ptr(), inc_arr.components
    temp = torch.empty(max(n * ar * inc_arr.components, 1), dtype=TORCH_DTYPES[inc_arr.elem_type], device=dev)
    _native.call("mp_exec_serial", L, off.data_ptr(), refs.data_ptr(), temp.data_ptr(), _native.stream_ptr())
    out = arrays[inc.array][0].cpu().numpy()
    return mesh.with_data(DataArray(inc_arr.name, inc_arr.set, inc_arr.components, out, arrays[inc.array][1]))

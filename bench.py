#!/usr/bin/env python
"""Benchmark: effective HBM GB/s and ms/iter of the indirect-increment loop,
hierarchical vs global colouring, on 1..8 B200s.

    python bench.py [--gpus N --steps K --warmup W --config C5 --reorder gps]
    python bench.py --impl reference        # the reference's CPU loop, same metric

Default workload (BASELINE.json configs[4], the 1/2/4/8-GPU config): the
Airfoil-style edge->cell flux loop on a 5657 x 5657 quad mesh (63,991,984
edges, 32,001,649 cells, fp64), hierarchical two-layer colouring (GPS
blocks, block size 128, the fastest measured schedule), values on the
1/1024 grid from a counter hash (synthetic).  ``roofline.frac`` is taken on
the consumed bytes of SURVEY 8(d) (``mp.consumed_bytes``: indirectly read
arrays counted only for the components the element function reads; C5's
equal the formula's, C4's are 1,915 MB of the formula's 3,387 MB);
``frac_strict`` also trims the direct arrays; ``value`` is the paper's
effective GB/s.  One step = one full execution of the loop over
the mesh.  Effective GB/s uses the paper's formula (simulator.py:315-328):
each array once, the incremented array twice, 4-byte mapping entries.
With N>1 GPUs the mesh is decomposed into x-slabs (owner compute; halo
import of q and export of increments through peer memory -- CUDA IPC
mailboxes, the export fused into the boundary blocks' write-back, each step
one CUDA graph; NCCL send/recv with --transport nccl); `value` is the
whole-mesh bytes over the max-over-ranks step time (strong scaling: the mesh
is fixed).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

#: default block layout per config (BASELINE.json configs): GPS for the 2D edge
#: loops, natural order for the hex node loop (GPS gives it 78 block colours,
#: SURVEY 8d), the reference's k-way partition for the face loop (the config
#: names k-way partitioned blocks; ~50 s to plan at 24M faces)
DEFAULT_REORDER = {"C1": "gps", "C2": "gps", "C3": "none", "C4": "partition", "C5": "gps"}
#: default block size per config (--block-size overrides): the k-way blocks of
#: the face loop at 256 faces (reuse 3.22 vs 2.92 at 128; pipelined-pull
#: 1.02 vs 1.08 ms, tools/gpu_c4bs.sh), 128 elsewhere
DEFAULT_BLOCK = {"C4": 256}
#: element orders of the global-colouring baseline timed beside the default
#: (GPS) one (global/none as well); the speed-up is also quoted
#: over the faster of the two
GLOBAL_COMPARE = {c: ("none",) for c in ("C1", "C2", "C3", "C4", "C5")}
#: other block layouts timed beside the headline (reported as vs_layout):
#: name -> (reorder, block size or None for --block-size, schedule(s) or None
#: for the headline's[, indirect-data layout, default --layout])
COMPARE_REORDER = {"C1": (("none", None, None), ("partition", None, None),  # hier/{none,gps,partition}
                          ("gps", 448, None), ("gps", 480, None)),                # and the paper's 448/480-element blocks
                   "C2": (("none", None, None),),
                   # the paper's handcrafted hex blocks (shape from tools/shape_sweep.sh),
                   # in AoS and in SoA (each consumed state / flux component a contiguous plane:
                   # 0.86 vs 0.93 ms, profiles/r02/c4_soa.log)
                   "C4": (("structured:4,4,8", 480, ("stream-pull", "pipelined", "pipelined-pull", "stream")),
                          ("structured:4,4,8", 480, ("stream-pull", "stream"), "soa"),
                          # the parallel GPU blocking (extension): same loop time as k-way, 1.2 s vs 21.6 s reorder
                          ("cluster", None, ("pipelined-pull", "stream-pull")))}
CONFIGS = {
    # name: (family, dims, kernel, dtype, staging)
    "C1": ("quad2d", (848, 848), "flux", "f64", "all-indirect"),
    "C2": ("tri2d", (1095, 1095), "flux", "f32", "all-indirect"),
    "C3": ("hex3d-nodes", (160, 160, 160), "scatter8", "f64", "all-indirect"),
    "C4": ("hex3d-faces", (200, 200, 200), "face-flux", "f64", "increment-only"),
    "C5": ("quad2d", (5657, 5657), "flux", "f64", "all-indirect"),
}
METRIC = "effective HBM GB/s and ms/iter per indirect loop vs global colouring, 1/2/4/8 GPU"
SCHEDULES = ("stream", "stream-pull", "stream-dataflow", "pipelined", "pipelined-pull", "colour", "dataflow")
L2_BYTES = 126 * 2**20
KERNEL_OF = {"stream": "hier_stream_kernel", "pipelined": "hier_pipe_kernel", "colour": "hier_block_kernel",
             "dataflow": "hier_block_kernel"}


def peaks():
    try:
        return json.loads((REPO / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def hbm_peak():
    p = peaks()
    if "hbm_gbs" in p:
        return float(p["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ----------------------------------------------------------------------------------
# clocks
# ----------------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index=0):
        self.rows = []
        self.proc = None
        self.dev = device_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 8 for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# ----------------------------------------------------------------------------------
# workload
# ----------------------------------------------------------------------------------


def quad_mesh(nx, ny, seed=0, xlo=0, xhi=None):
    """Full (or x-slab) quad mesh with hashed 1/1024-grid values (synthetic)."""
    import torch

    import paper_1802_03749_b200 as mp
    from paper_1802_03749_b200.workloads import hashed_grid_values, quad2d_table

    table, gids = quad2d_table(nx, ny, xlo, xhi)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    cells_used = np.unique(table) if (xlo != 0 or (xhi is not None and xhi != nx)) else None
    ncell = nx * ny
    if cells_used is None:
        cid = torch.arange(ncell, dtype=torch.int64, device=dev)
        local_table = table
    else:
        cid = torch.as_tensor(cells_used, device=dev)
        local_table = np.searchsorted(cells_used, table)
    q = hashed_grid_values(cid[:, None] * 4 + torch.arange(4, device=dev), seed, 1).cpu().numpy()
    g = torch.as_tensor(gids, device=dev)
    w = hashed_grid_values(g[:, None] * 2 + torch.arange(2, device=dev), seed, 3).cpu().numpy()
    edges = mp.MeshSet("edges", local_table.shape[0])
    cells = mp.MeshSet("cells", cid.numel())
    data = [mp.DataArray("q", cells, 4, q.reshape(-1)), mp.DataArray("res", cells, 4, np.zeros(cid.numel() * 4)),
            mp.DataArray("w", edges, 2, w.reshape(-1))]
    mesh = mp.Mesh.build([edges, cells], [mp.Mapping("e2c", edges, cells, local_table)], data,
                         {"family": "quad2d", "dims": f"{nx} {ny}", "seed": str(seed), "dtype": "f64"})
    return mesh, (None if cells_used is None else cells_used)


def make_mesh(cfg_name, seed=0):
    import paper_1802_03749_b200 as mp
    from paper_1802_03749_b200 import workloads

    family, dims, kname, dtype, staging = CONFIGS[cfg_name]
    if family == "quad2d":
        mesh, _ = quad_mesh(*dims, seed=seed)
    else:
        mesh = workloads.generate_mesh(family, dims, seed=seed, dtype=dtype, arrays=workloads.arrays_for_kernel(kname))
    return mesh, mp.kernel_for_mesh(kname, mesh), staging


# ----------------------------------------------------------------------------------
# timing
# ----------------------------------------------------------------------------------


class L2Flusher:
    def __init__(self, needed):
        import torch

        self.buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device="cuda") if needed else None

    def __call__(self):
        if self.buf is not None:
            self.buf.add_(1)


def time_steps(step, K, W, flush, stream=None):
    """Per-step CUDA-event times (ms) on the launching stream, L2 flushed
    between steps when the working set fits in L2."""
    import torch

    for _ in range(W):
        flush()
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, b in evs:
        flush()
        a.record()
        step()
        b.record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def kernel_share(step, K):
    """Average device duration of the launches inside one step (CUDA events
    around the hot kernel launches only); for the dataflow schedule this is
    the single executor kernel."""
    import torch

    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        step()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


def _reference_package():
    """The unmodified reference package, pip-installed into baseline/_ref
    (tools/stage_reference.sh; git-ignored, travels with the snapshot), or None."""
    ref = REPO / "baseline" / "_ref"
    if not (ref / "meshplan" / "__init__.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import meshplan

        return meshplan
    except Exception:  # pragma: no cover - a broken install falls back to the port
        return None


def _sample(mesh, kernel_name, max_edges):
    """The first ``max_edges`` elements of the loop with the points they use
    (renumbered densely, order kept): a bounded sample of the same workload."""
    m = next(iter(mesh.mappings.values()))
    n = min(m.from_set.size, max_edges)
    table = m.table[:n]
    used = np.unique(table)
    local = np.searchsorted(used, table)
    read = {"flux": "q", "face-flux": "state", "face-flux-heavy": "state"}.get(kernel_name)
    direct = {"flux": "w", "flux-noread": "w", "scatter8": "stress"}.get(kernel_name, "facew")
    inc = {"flux": "res", "flux-noread": "res", "scatter8": "force"}.get(kernel_name, "flux")
    arrays = {inc: np.ascontiguousarray(mesh.data[inc].view2d()[used]),
              direct: np.ascontiguousarray(mesh.data[direct].view2d()[:n])}
    if read is not None:
        arrays[read] = np.ascontiguousarray(mesh.data[read].view2d()[used])
    return m, n, used, local, read, direct, inc, arrays


def cpu_runner(mesh, kernel_name, max_edges=4_000_000):
    """The reference's CPU loop on a bounded sample of the workload, on this
    host: the UNMODIFIED reference ``meshplan.execute_serial``
    (simulator.py:215-230, numpy; single-threaded) from baseline/_ref when
    installed (kind "reference"), else its restatement in oracle/loops.py
    (kind "port").  Returns (run, useful bytes of the sample by the paper
    formula, kind, description)."""
    m, n, used, local, read, direct, inc, arrays = _sample(mesh, kernel_name, max_edges)
    ref = _reference_package()
    if ref is not None:
        from meshplan.bench_kernels import kernel_for_mesh as ref_kernel_for_mesh

        fr, to = ref.MeshSet(m.from_set.name, n), ref.MeshSet(m.to_set.name, used.size)
        sets = {m.from_set.name: fr, m.to_set.name: to}
        data = [ref.DataArray(name, to if name != direct else fr, a.shape[1], a.ravel(), "aos")
                for name, a in arrays.items()]
        rmesh = ref.Mesh.build([fr, to], [ref.Mapping(m.name, fr, to, local.astype(np.int64))], data,
                               dict(mesh.meta))
        kern = ref_kernel_for_mesh(kernel_name, rmesh)
        ub = int(ref.simulator._useful_bytes(kern, rmesh))
        run = lambda: ref.execute_serial(rmesh, kern)  # noqa: E731
        kind, what = "reference", "meshplan.execute_serial (the unmodified reference, baseline/_ref, numpy backend)"
        del sets
    else:
        from oracle import loops

        arr = [(used.size, arrays[inc].shape[1], arrays[inc].itemsize, True),
               (n, arrays[direct].shape[1], arrays[direct].itemsize, False)]
        if read is not None:
            arr.append((used.size, arrays[read].shape[1], arrays[read].itemsize, False))
        ub = loops.useful_bytes(n, m.arity, arr)
        run = lambda: loops.serial_loop(kernel_name, local, arrays.get(read), arrays[direct], arrays[inc])  # noqa
        kind, what = "port", "execute_serial restated in numpy (oracle/loops.py)"
    desc = f"{what} on the first {n} of {m.from_set.size} elements ({used.size} points)"
    return run, ub, kind, desc


def cpu_baseline(mesh, kernel_name, seconds=10.0, max_edges=4_000_000):
    """``cpu_runner``'s loop timed for about ``seconds`` (at least 3 runs)."""
    run, ub, kind, desc = cpu_runner(mesh, kernel_name, max_edges)
    times = []
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or len(times) < 3:
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return {"value": round(ub / t / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": kind,
            "sample": f"{desc}, median of {len(times)} runs, {t * 1e3:.1f} ms/run; host has {os.cpu_count()} cores, "
                      "the reference loop is single-threaded numpy",
            "ms_per_run": round(t * 1e3, 3), "useful_bytes": ub}


# ----------------------------------------------------------------------------------
# arms
# ----------------------------------------------------------------------------------


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    mesh, kernel, _ = make_mesh(args.config)
    family, dims, kname, dtype, _ = CONFIGS[args.config]
    run, ub, kind, desc = cpu_runner(mesh, kname)
    del mesh, kernel
    per_step = []
    for i in range(args.warmup + args.steps):  # W untimed, then K timed runs of the bounded sample
        t0 = time.perf_counter()
        run()
        if i >= args.warmup:
            per_step.append((time.perf_counter() - t0) * 1e3)
    ms = statistics.median(per_step)
    val = round(ub / (ms * 1e-3) / 1e9, 4)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "config": {"workload": f"{args.config} {family} {'x'.join(map(str, dims))} {kname} {dtype} "
                               "(bounded sample, see cpu_baseline.sample)"},
        "cpu_baseline": {"value": val, "unit": "GB/s", "cores": 1, "kind": kind,
                         "sample": f"{desc}, median of {len(per_step)} runs, {ms:.1f} ms/run; host has "
                                   f"{os.cpu_count()} cores, the reference loop is single-threaded numpy"},
        "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def verify_full(hier, glob, kernel, main, gl):
    """Results of one loop execution at the full config, bit for bit: the
    headline hierarchical loop == global colouring == the device serial loop
    (element order, simulator.py:215-230), restored to the original numbering
    (the hashed 1/1024-grid data makes every sum exact, so any correct order
    agrees; tests/test_gpu_configs.py pins the serial loop to the reference's
    own result at these sizes by CRC)."""
    import torch

    import paper_1802_03749_b200 as mp

    inc = next(a.array for a in kernel.args if a.mode == "increment")

    def once(loop, plan):
        t = loop.tensors[inc]
        saved = t.clone()
        t.zero_()
        loop.run()
        torch.cuda.synchronize()
        got = t.cpu().numpy().copy()
        t.copy_(saved)
        arr = plan.mesh.data[inc]
        res = plan.restore_data(plan.mesh.with_data(mp.DataArray(arr.name, arr.set, arr.components, got,
                                                                 arr.layout)))
        return np.ascontiguousarray(res.data[inc].view2d())

    serial = mp.bind(hier, kernel, schedule="temp-array")
    want = once(serial, hier)
    del serial
    h = once(main, hier)
    g = once(gl, glob)
    ok_h = bool(np.array_equal(h.view(np.uint8), want.view(np.uint8)))
    ok_g = bool(np.array_equal(g.view(np.uint8), want.view(np.uint8)))
    return {"checked": "one execution from zeroed increments, restored numbering: headline hierarchical == "
                       "global colouring == device serial loop (element order), bit for bit",
            "hier_equals_serial": ok_h, "global_equals_serial": ok_g,
            "nonzero_rows": int(np.count_nonzero(np.any(want != 0, axis=1)))}


def reference_plan_times(args):
    """The reference planner's wall time for the same plans (next
    to the GPU plan-build times), as recorded by tests/golden/make_fingerprints.py
    when it ran the real reference at these sizes (8-core build container,
    numba backend); None where it was not run."""
    try:
        fp = json.loads((REPO / "tests" / "golden" / "fingerprints.json").read_text())
    except (OSError, ValueError):
        return None
    name = args.config if args.block_size == 128 else f"{args.config}k{args.block_size}"
    plans = fp.get(name, {}).get("plans", {})
    out = {k: v.get("build_s") for k, v in plans.items()
           if k in (f"hier/{args.reorder}", f"global/{args.global_reorder}")}
    return out or None


def our_arm(args):
    import torch

    import paper_1802_03749_b200 as mp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        from paper_1802_03749_b200 import decomp

        return decomp.bench_rank(args, rank, world)
    torch.cuda.set_device(0)
    family, dims, kname, dtype, staging = CONFIGS[args.config]
    t0 = time.perf_counter()
    mesh, kernel, staging = make_mesh(args.config)
    t_gen = time.perf_counter() - t0
    ub = mp.useful_bytes(kernel, mesh)
    cb = mp.consumed_bytes(kernel, mesh)
    cb_strict = mp.consumed_bytes(kernel, mesh, strict=True)
    flush = L2Flusher(ub < 2 * L2_BYTES)

    results = {}
    plans = {}
    t0 = time.perf_counter()
    hier = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(
        reorder=args.reorder, layout=args.layout, staging=staging, block_size=args.block_size))
    t_plan_h = time.perf_counter() - t0
    plans["hier"] = hier
    sampler = ClockSampler()
    sampler.start()
    loops = {}
    for sched in SCHEDULES:
        lp = mp.bind(hier, kernel, schedule=sched)
        loops[sched] = lp
        times = time_steps(lp.run, args.steps, args.warmup, flush)
        results[f"hier_{sched}"] = times
    if args.schedule == "best":
        args.schedule = min(SCHEDULES, key=lambda sc: statistics.median(results[f"hier_{sc}"]))
    # the headline schedule's launches captured as one CUDA graph (colour
    # schedules; the same kernels, one submission per loop)
    graph = None
    if "dataflow" not in args.schedule:
        graph = loops[args.schedule].capture()
        results["graph"] = time_steps(graph.replay, args.steps, args.warmup, flush)
    clocks = sampler.stop()

    t0 = time.perf_counter()
    glob = mp.build_global_plan(mesh, kernel, mp.PlanConfig(strategy="global", reorder=args.global_reorder,
                                                              layout=args.layout, block_size=args.block_size))
    t_plan_g = time.perf_counter() - t0
    gl = mp.bind(glob, kernel)
    results["global"] = time_steps(gl.run, args.steps, args.warmup, flush)
    # atomics baseline (the paper's other race-avoidance strategy) on the same
    # element order and layout as the hierarchical plan
    results["atomic"] = time_steps(mp.bind(hier, kernel, schedule="atomic").run, args.steps, args.warmup, flush)
    # and the temporary-array strategy (per-(element, slot) temps + per-point
    # fold in element order: the serial loop's result, bit for bit)
    tmp_loop = mp.bind(hier, kernel, schedule="temp-array")
    results["temp_array"] = time_steps(tmp_loop.run, args.steps, args.warmup, flush)
    del tmp_loop

    # the configs that compare block layouts (BASELINE.json configs[1]: natural
    # vs GPS-reordered) time the other layout with the headline schedule too
    vs_layout = {}
    global_by_reorder = {}
    for other in GLOBAL_COMPARE.get(args.config, ()):
        if other == args.global_reorder:
            continue
        g_alt = mp.build_global_plan(mesh, kernel, mp.PlanConfig(strategy="global", reorder=other, layout=args.layout,
                                                                   block_size=args.block_size))
        ms_g = statistics.median(time_steps(mp.bind(g_alt, kernel).run, args.steps, args.warmup, flush))
        global_by_reorder[other] = {"ms_per_step": round(ms_g, 5), "colours": g_alt.num_colours}
        del g_alt
    for other, bs, sched, *lay in COMPARE_REORDER.get(args.config, ()):
        lay = lay[0] if lay else args.layout
        if other == args.reorder and lay == args.layout and (bs or args.block_size) == args.block_size:
            continue
        t0 = time.perf_counter()
        alt = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(
            reorder=other, layout=lay, staging=staging, block_size=bs or args.block_size))
        t_alt = time.perf_counter() - t0
        by_sched = {}
        for sc in (sched if isinstance(sched, tuple) else (sched or args.schedule,)):
            alt_loop = mp.bind(alt, kernel, schedule=sc)
            by_sched[sc] = statistics.median(time_steps(alt_loop.run, args.steps, args.warmup, flush))
            del alt_loop
        sc = min(by_sched, key=by_sched.get)
        ms_alt = by_sched[sc]
        key = other + ("" if lay == args.layout else f"/{lay}") + (f"@{bs}" if bs and other == args.reorder else "")
        vs_layout[key] = {"ms_per_step": round(ms_alt, 5), "gbps": round(ub / (ms_alt * 1e-3) / 1e9, 2),
                            "frac": round(cb / (ms_alt * 1e-3) / 1e9 / hbm_peak()[0], 4),
                            "frac_formula": round(ub / (ms_alt * 1e-3) / 1e9 / hbm_peak()[0], 4),
                            "block_size": bs or args.block_size, "schedule": sc, "layout": lay,
                            "ms_by_schedule": {k: round(v, 5) for k, v in by_sched.items()},
                            "reuse_factor": round(mp.reuse_factor(alt), 4),
                            "block_colours": alt.block_colours.num_colours, "plan_build_s": round(t_alt, 2)}
        del alt
    # parity self-check at the full config (outside the timed regions): one
    # execution of the headline loop, of global colouring and of the device
    # serial loop (temp-array strategy: per-point fold in element order, the
    # reference execute_serial's np.add.at order), each from zeroed increments
    main = loops[args.schedule]
    parity = verify_full(hier, glob, kernel, main, gl)

    # end to end through the public API with host buffers (pinned), H2D + D2H in the region
    inputs = {a.array: hier.mesh.data[a.array].values for a in kernel.args}
    inc_name = next(a.array for a in kernel.args if a.mode == "increment")
    out = torch.empty(hier.mesh.data[inc_name].values.size, dtype=main.tensors[inc_name].dtype, pin_memory=True)
    h2d = sum(v.nbytes for v in inputs.values())
    d2h = out.numel() * out.element_size()

    def e2e_step():
        main.run_host(inputs, out)

    n_e2e = max(3, args.steps // 2)
    e2e_serial = time_steps(e2e_step, n_e2e, args.warmup, flush)
    # the same steps streamed (mp.HostStream: two streams and device array
    # sets, so step k's D2H overlaps step k+1's H2D and compute); every step
    # still copies its inputs in and its result out inside the timed region
    hs = mp.HostStream(hier, kernel, schedule=args.schedule, depth=2)
    outs = [out, torch.empty_like(out, pin_memory=True)]
    for k in range(args.warmup):
        hs.step(inputs, outs[k % 2])
    hs.synchronize()
    torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record()
    hs.wait_on(ea)
    for k in range(n_e2e):
        hs.step(inputs, outs[k % 2])
    hs.join()
    eb.record()
    torch.cuda.synchronize()
    e2e_ms = ea.elapsed_time(eb) / n_e2e
    del hs

    ms_direct = statistics.median(results[f"hier_{args.schedule}"])
    ms_graph = statistics.median(results["graph"]) if "graph" in results else None
    use_graph = ms_graph is not None and ms_graph < ms_direct
    ms = ms_graph if use_graph else ms_direct
    ms_glob = statistics.median(results["global"])
    per_schedule = {s: round(statistics.median(results[f"hier_{s}"]), 5) for s in SCHEDULES}
    gbps = ub / (ms * 1e-3) / 1e9
    peak, peak_kind = hbm_peak()
    launches = main.launches_per_run()
    cpu = cpu_baseline(mesh, kname, seconds=args.cpu_seconds) if args.cpu_seconds > 0 else None
    traffic = None
    prof = REPO / "profiles" / "traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(f"{args.config}:{args.reorder}:{args.schedule}")  # per step
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": round(gbps, 2), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "config": {
            "workload": f"{args.config}: {family} {'x'.join(map(str, dims))} {kname} {dtype}, "
                        f"{mesh.sets[kernel.iter_set_name(mesh)].size} elements",
            "strategy": "hier", "reorder": args.reorder, "layout": args.layout, "staging": staging,
            "block_size": args.block_size, "schedule": args.schedule,
            "staged_rows": ("read and increment rows (all indirect data through shared memory)"
                            if hier._device.stage_reads else "increment rows only (reads from global)"),
            "submission": "CUDA graph of the loop's launches" if use_graph else "direct launches",
            "l2": "flushed between steps" if flush.buf is not None else "inputs larger than L2 (no flush)",
            "useful_bytes_per_step": ub, "parallelism": "single GPU",
        },
        "vs_global": {
            "global_ms": round(ms_glob, 5), "global_gbps": round(ub / (ms_glob * 1e-3) / 1e9, 2),
            "global_reorder": args.global_reorder, "global_colours": glob.num_colours,
            "global_other_orders": global_by_reorder or None,
            "speedup_hier_over_best_global": round(min([ms_glob] + [v["ms_per_step"] for v in global_by_reorder.values()]) / ms, 3),
            "hier_ms_by_schedule": per_schedule,
            "headline_direct_ms": round(ms_direct, 5),
            "headline_graph_ms": None if ms_graph is None else round(ms_graph, 5),
            "speedup_hier_over_global": round(ms_glob / ms, 3),
            "atomic_ms": round(statistics.median(results["atomic"]), 5),
            "speedup_hier_over_atomic": round(statistics.median(results["atomic"]) / ms, 3),
            "temp_array_ms": round(statistics.median(results["temp_array"]), 5),
            "speedup_hier_over_temp_array": round(statistics.median(results["temp_array"]) / ms, 3),
            "block_colours": hier.block_colours.num_colours, "num_blocks": hier.num_blocks,
            "reuse_factor": round(mp.reuse_factor(hier), 4),
            "thread_colours_mean": round(float(hier.thread_colour_counts.mean()), 3),
        },
        "vs_layout": vs_layout or None,
        "roofline": {"bound": "hbm", "achieved": round(cb / (ms * 1e-3) / 1e9, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(cb / (ms * 1e-3) / 1e9 / peak, 4), "traffic": traffic, "peak_kind": peak_kind,
                     "bytes": "consumed (SURVEY 8(d)): indirectly read arrays only the components the element "
                              "function reads, every row once; direct arrays whole; increments read+written "
                              "once; 4-byte map entries",
                     "consumed_bytes_per_step": cb,
                     "frac_strict": round(cb_strict / (ms * 1e-3) / 1e9 / peak, 4),
                     "strict_bytes_per_step": cb_strict,
                     "achieved_formula": round(gbps, 2), "frac_formula": round(gbps / peak, 4),
                     "formula_bytes_per_step": ub,
                     "traffic_over_consumed": None if not traffic else round(traffic / cb, 3),
                     "kernel": f"{KERNEL_OF[args.schedule.split('-')[0]]} "
                               f"({args.schedule} schedule, {launches} launch(es)/step; achieved = consumed "
                               f"bytes / summed device time of the step's launches)"},
        "e2e": {"value": round(ub / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": round(e2e_ms, 3),
                "serial_ms_per_step": round(statistics.median(e2e_serial), 3),
                "path": "mp.HostStream (public API): per step pinned host arrays -> H2D -> executor -> D2H, "
                        "consecutive steps on two streams with their own device arrays (serial_ms_per_step: "
                        "DeviceLoop.run_host one step at a time)"},
        "parity": parity,
        "gpu_launches": int(launches * args.steps),
        "clocks": clocks,
        "cpu_baseline": cpu,
        "plan_build_s": {"generate": round(t_gen, 2), "hier": round(t_plan_h, 2), "global": round(t_plan_g, 2),
                         "reference": reference_plan_times(args)},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--reorder", default=None, help="block layout (default: per config, DEFAULT_REORDER)")
    ap.add_argument("--global-reorder", default="gps")
    ap.add_argument("--layout", default="aos")
    ap.add_argument("--block-size", type=int, default=None)
    ap.add_argument("--schedule", default="best", choices=SCHEDULES + ("best",),
                    help="headline executor schedule; 'best' = fastest of the measured schedules")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--transport", default="peer", choices=("peer", "nccl"),
                    help="N>1 halo exchange: peer-memory puts (graph-captured steps) or NCCL send/recv")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.reorder is None:
        args.reorder = DEFAULT_REORDER[args.config]
    if args.block_size is None:
        args.block_size = DEFAULT_BLOCK.get(args.config, 128)
    if args.impl == "reference":
        return reference_arm(args)
    return our_arm(args)


if __name__ == "__main__":
    sys.exit(main())

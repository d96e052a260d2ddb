"""GPU parity: the sm_100a planner and executors against the reference.

Golden vectors come from the real reference (tests/golden/make_golden.py);
the oracle (oracle/, itself pinned by test_oracle_golden.py) checks sizes
without fixtures.  Everything here calls through the C ABI.
"""

import dataclasses

import numpy as np
import pytest
import torch

import paper_1802_03749_b200 as mp
from conftest import INC_OF, bit_equal, case_mesh, golden_cases, load_case
from helpers import config_of, reference_plan

pytestmark = pytest.mark.gpu

CASES = golden_cases()
SCHEDULES = ("dataflow", "colour", "pipelined", "pipelined-dataflow", "pipelined-pull", "pipelined-dataflow-pull",
             "stream", "stream-dataflow", "stream-pull")


def _ids(c):
    return f"{c['file']}-{c['family']}-{c['kernel']}-{c['dtype']}-{c['strategy']}-{c['reorder']}"


def _build(rec, mesh, kernel):
    cfg = config_of(rec)
    if rec["strategy"] == "global":
        return mp.build_global_plan(mesh, kernel, cfg)
    return mp.build_hierarchical_plan(mesh, kernel, cfg)


def _run(plan, kernel, schedule="dataflow"):
    if isinstance(plan, mp.GlobalPlan):
        return mp.execute_global(plan, kernel)
    return mp.execute_hierarchical(plan, kernel, schedule=schedule)


def _v2(mesh, name):
    return np.ascontiguousarray(mesh.data[name].view2d())


# ---- executors on the reference's own plans (covers every reorder mode) -------------


@pytest.mark.parametrize("rec", CASES, ids=_ids)
def test_executor_on_reference_plan_bit_exact(rec):
    z = load_case(rec)
    rmesh = case_mesh(rec, random=True, arrays=z)
    kernel = mp.kernel_for_mesh(rec["kernel"], rmesh)
    plan = reference_plan(rec, z, rmesh, kernel)
    for sched in (SCHEDULES if rec["strategy"] == "hier" else ("-",)):
        res, rep = _run(plan, kernel, sched)
        assert bit_equal(_v2(res, INC_OF[rec["kernel"]]), z["rand_exec_inc"]), sched
        if rec["strategy"] == "hier":
            assert np.array_equal(rep.sync_counts, plan.thread_colour_counts + 2)


# ---- planner parity (bit-exact plans) --------------------------------------------------


PLANNED = CASES  # none, gps, partition (k-way) and structured plans


@pytest.mark.parametrize("rec", PLANNED, ids=_ids)
def test_gpu_planner_matches_reference(rec):
    z = load_case(rec)
    mesh = case_mesh(rec)
    kernel = mp.kernel_for_mesh(rec["kernel"], mesh)
    plan = _build(rec, mesh, kernel)
    m = next(iter(mesh.mappings.values()))
    assert np.array_equal(plan.set_perms[m.from_set.name].forward, z["elem_fwd"])
    assert np.array_equal(plan.set_perms[m.to_set.name].forward, z["point_fwd"])
    assert np.array_equal(plan.mesh.mappings[m.name].table, z["plan_table"])
    if rec["strategy"] == "global":
        assert np.array_equal(plan.colour_offsets, z["colour_offsets"])
        assert np.array_equal(plan.colours.colours, z["colours"])
    else:
        assert np.array_equal(plan.block_offsets, z["block_offsets"])
        assert np.array_equal(plan.block_colours.colours, z["block_colours"])
        assert np.array_equal(plan.thread_colours, z["thread_colours"])
        assert np.array_equal(plan.thread_colour_counts, z["thread_colour_counts"])
        ((_, (sp, si)),) = plan.staged.items()
        ((_, (wp, wi)),) = plan.written.items()
        assert np.array_equal(sp, z["staged_ptr"]) and np.array_equal(si, z["staged_ids"])
        assert np.array_equal(wp, z["written_ptr"]) and np.array_equal(wi, z["written_ids"])
        assert np.array_equal(plan.shared_bytes, z["shared_bytes"])
        assert mp.reuse_factor(plan) == pytest.approx(rec["reuse_factor"], abs=1e-12)
    # and the whole pipeline: plan -> execute -> restore == reference serial (exact data)
    res, _ = _run(plan, kernel)
    restored = plan.restore_data(res)
    got = _v2(restored, INC_OF[rec["kernel"]])
    if rec["kernel"] == "face-flux-heavy":  # sqrt scaling is not on the 1/1024 grid: reordered sums round
        assert_close(got, z["serial_inc"], rel=1e-12 if rec["dtype"] == "f64" else 1e-6)
    else:
        assert bit_equal(got, z["serial_inc"])


def assert_close(a, b, rel):
    """The reference's _verify rule (cli.py:161-188): |a-b| <= rel * max(|a|, |b|, max|b|)."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), np.abs(b).max(initial=0.0))
    assert np.all(np.abs(a - b) <= rel * scale)


# ---- serial-order executor ---------------------------------------------------------------


@pytest.mark.parametrize("rec", [c for c in CASES if c["strategy"] == "global" and c["reorder"] == "none"], ids=_ids)
def test_gpu_serial_bit_exact(rec):
    z = load_case(rec)
    mesh = case_mesh(rec)
    kernel = mp.kernel_for_mesh(rec["kernel"], mesh)
    assert bit_equal(_v2(mp.execute_serial(mesh, kernel), INC_OF[rec["kernel"]]), z["serial_inc"])
    rmesh = case_mesh(rec, random=True, arrays=z)
    assert bit_equal(_v2(mp.execute_serial(rmesh, kernel), INC_OF[rec["kernel"]]), z["rand_serial_inc"])


# ---- checks before any output (mutation tests, test_simulator.py:82-198) ----------------


def _flux_plan(strategy, reorder="none", bs=16, dims=(8, 8)):
    mesh = mp.generate_mesh("quad2d", dims, dtype="i64")
    kernel = mp.kernel_for_mesh("flux", mesh)
    cfg = mp.PlanConfig(strategy=strategy, reorder=reorder, block_size=bs)
    build = mp.build_global_plan if strategy == "global" else mp.build_hierarchical_plan
    return build(mesh, kernel, cfg), kernel


def test_corrupted_global_colours_race():
    plan, kernel = _flux_plan("global", dims=(4, 4))
    off = plan.colour_offsets.copy()
    off[1:] = off[-1]
    bad = dataclasses.replace(plan, colour_offsets=off,
                              colours=mp.ColourAssignment.from_colours(np.zeros(len(plan.colours.colours), np.int64)))
    with pytest.raises(mp.RaceError, match=r"elements \d+ and \d+"):
        mp.execute_global(bad, kernel)


def test_corrupted_thread_colours_race():
    plan, kernel = _flux_plan("hier", bs=32)
    tc = plan.thread_colours.copy()
    b = int(np.argmax(plan.thread_colour_counts))
    lo, hi = plan.block_range(b)
    tc[lo:hi] = 0
    with pytest.raises(mp.RaceError, match="thread colouring"):
        mp.execute_hierarchical(dataclasses.replace(plan, thread_colours=tc), kernel)


def test_corrupted_block_colours_race():
    plan, kernel = _flux_plan("hier", bs=16)
    assert plan.block_colours.num_colours > 1
    bad = dataclasses.replace(plan, block_colours=mp.ColourAssignment.from_colours(np.zeros(plan.num_blocks, np.int64)))
    with pytest.raises(mp.RaceError, match="block colouring"):
        mp.execute_hierarchical(bad, kernel)


def test_staged_miss_is_capacity_fault():
    plan, kernel = _flux_plan("hier", bs=16, dims=(6, 6))
    indptr, ids = plan.staged["cells"]
    truncated = {"cells": (indptr - np.arange(len(indptr)), ids[: -(len(indptr) - 1)])}
    with pytest.raises(mp.CapacityError):
        mp.execute_hierarchical(dataclasses.replace(plan, staged=truncated), kernel)


def test_shared_capacity_fault_names_block():
    mesh = mp.generate_mesh("hex3d-faces", (6, 6, 6), dtype="f64")
    kernel = mp.kernel_for_mesh("face-flux", mesh)
    hw = dataclasses.replace(mp.P100, shared_bytes_per_sm=1024)
    with pytest.raises(mp.CapacityError, match=r"block \d+ needs \d+ shared bytes"):
        mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(block_size=128), hw)


def test_unknown_kernel_has_no_fallback():
    mesh = mp.generate_mesh("quad2d", (4, 4))
    k = mp.kernel_for_mesh("flux", mesh)
    plan = mp.build_hierarchical_plan(mesh, k)
    custom = dataclasses.replace(k, device_op=None)
    with pytest.raises(mp.KernelSpecError, match="no device functor"):
        mp.execute_hierarchical(plan, custom)


# ---- larger meshes: size-independent properties ---------------------------------------


@pytest.mark.parametrize("family,dims,kname", [
    ("quad2d", (256, 192), "flux"),
    ("tri2d", (160, 150), "flux"),
    ("hex3d-nodes", (24, 20, 16), "scatter8"),
    ("hex3d-faces", (20, 18, 16), "face-flux"),
])
def test_medium_meshes_all_strategies_exact(family, dims, kname):
    """Quantised data: every strategy / schedule equals the GPU serial
    executor and the oracle, bit for bit; unit increments count incidence."""
    from oracle import loops

    mesh = mp.generate_mesh(family, dims, dtype="f64")
    kernel = mp.kernel_for_mesh(kname, mesh)
    inc = INC_OF[kname]
    m = next(iter(mesh.mappings.values()))
    read = {"flux": "q", "face-flux": "state"}.get(kname)
    direct = {"flux": "w", "scatter8": "stress", "face-flux": "facew"}[kname]
    want = loops.serial_loop(kname, m.table, None if read is None else mesh.data[read].view2d(),
                             np.ascontiguousarray(mesh.data[direct].view2d()), _v2(mesh, inc))
    assert bit_equal(_v2(mp.execute_serial(mesh, kernel), inc), want)
    staging = "increment-only" if kname == "face-flux" else "all-indirect"
    for strategy, reorder, layout in (("global", "none", "aos"), ("global", "gps", "soa"), ("hier", "none", "soa"),
                                      ("hier", "gps", "aos")):
        cfg = mp.PlanConfig(strategy=strategy, reorder=reorder, layout=layout, staging=staging)
        plan = (mp.build_global_plan if strategy == "global" else mp.build_hierarchical_plan)(mesh, kernel, cfg)
        for sched in (SCHEDULES if strategy == "hier" else ("-",)):
            res, _ = _run(plan, kernel, sched)
            assert bit_equal(_v2(plan.restore_data(res), inc), want), (strategy, reorder, sched)
    unit = mp.kernel_for_mesh(kname, mesh, unit=True)
    plan = mp.build_hierarchical_plan(mesh, unit, mp.PlanConfig(reorder="gps"))
    res, _ = mp.execute_hierarchical(plan, unit)
    got = _v2(plan.restore_data(res), inc)
    counts = np.bincount(m.table.ravel(), minlength=m.to_set.size).astype(got.dtype)
    assert np.array_equal(got, counts[:, None] * np.ones((1, got.shape[1]), dtype=got.dtype))


@pytest.mark.parametrize("family,dims,kname,bs", [
    ("quad2d", (96, 80), "flux", 128),
    ("tri2d", (60, 50), "flux", 96),
    ("hex3d-nodes", (12, 10, 14), "scatter8", 128),
    ("hex3d-faces", (10, 9, 8), "face-flux", 64),
])
def test_cluster_reorder_plans_are_valid_and_exact(family, dims, kname, bs):
    """The GPU clustering blocking (extension): widths <= S, race-free (checked
    on execute), every schedule exact vs serial, reuse at least GPS's."""
    from oracle import loops

    mesh = mp.generate_mesh(family, dims, dtype="i64")
    kernel = mp.kernel_for_mesh(kname, mesh)
    inc = INC_OF[kname]
    m = next(iter(mesh.mappings.values()))
    read = {"flux": "q", "face-flux": "state"}.get(kname)
    direct = {"flux": "w", "scatter8": "stress", "face-flux": "facew"}[kname]
    want = loops.serial_loop(kname, m.table, None if read is None else mesh.data[read].view2d(),
                             np.ascontiguousarray(mesh.data[direct].view2d()), _v2(mesh, inc))
    staging = "increment-only" if kname == "face-flux" else "all-indirect"
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="cluster", block_size=bs, staging=staging))
    assert plan.working_threads().max() <= bs
    for sched in SCHEDULES:
        res, _ = mp.execute_hierarchical(plan, kernel, schedule=sched)
        assert np.array_equal(_v2(plan.restore_data(res), inc), want), sched
    gps = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps", block_size=bs, staging=staging))
    assert mp.reuse_factor(plan) >= 0.95 * mp.reuse_factor(gps)


def test_dataflow_repeated_runs_accumulate_exactly():
    """Epoch-stamped flags: many back-to-back dataflow runs stay exact."""
    mesh = mp.generate_mesh("quad2d", (128, 100), dtype="f64")
    kernel = mp.kernel_for_mesh("flux", mesh)
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps"))
    loops = [mp.bind(plan, kernel, schedule=s) for s in SCHEDULES]
    for _ in range(7):
        for lp in loops:
            lp.run()
    torch.cuda.synchronize()
    for lp in loops[1:]:
        assert torch.equal(loops[0].tensors["res"], lp.tensors["res"])


@pytest.mark.parametrize("family,dims,kname,reorder,bs", [
    ("quad2d", (700, 640), "flux", "gps", 128),
    ("quad2d", (300, 280), "flux", "none", 256),
    ("tri2d", (400, 380), "flux", "gps", 128),
    ("hex3d-nodes", (40, 36, 30), "scatter8", "none", 128),
    ("hex3d-faces", (40, 36, 30), "face-flux", "gps", 128),
])
def test_schedules_agree_on_random_data_many_blocks(family, dims, kname, reorder, bs):
    """Random (non-quantised) data, thousands of blocks per launch and several
    back-to-back runs: every schedule applies each point's writers in the same
    order, so all results are bit-identical to the paper's colour schedule
    (exercises the dataflow readiness / late paths and multi-row threads)."""
    mesh = mp.generate_mesh(family, dims, dtype="f64")
    kernel = mp.kernel_for_mesh(kname, mesh)
    staging = "increment-only" if kname == "face-flux" else "all-indirect"
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder=reorder, block_size=bs, staging=staging))
    g = torch.Generator(device="cuda").manual_seed(7)
    base = {}
    for a in kernel.args:
        if a.array not in base:
            n = plan.mesh.data[a.array].values.size
            base[a.array] = torch.rand(n, generator=g, device="cuda", dtype=torch.float64) * 2 - 1
    inc = INC_OF[kname]
    out = {}
    for sched in SCHEDULES:
        t = {k: v.clone() for k, v in base.items()}
        lp = mp.bind(plan, kernel, tensors=t, schedule=sched)
        for _ in range(3):
            lp.run()
        torch.cuda.synchronize()
        out[sched] = t[inc].cpu().numpy()
    for sched in SCHEDULES:
        assert bit_equal(out[sched], out["colour"]), sched


def test_stream_tma_gather_variant_matches_colour_schedule():
    """The opt-in TMA gather4 variant of the streamed executor (read rows
    through the tensor engine, MESHPLAN_STREAM_TMA=1, read once per process)
    gives the same bits as the warp-specialised and CTA-per-block executors."""
    import subprocess
    import sys
    import textwrap
    from pathlib import Path

    code = textwrap.dedent("""
        import numpy as np, torch, paper_1802_03749_b200 as mp
        mesh = mp.generate_mesh("quad2d", (300, 260), dtype="f64")
        kernel = mp.kernel_for_mesh("flux", mesh)
        plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps"))
        g = torch.Generator(device="cuda").manual_seed(3)
        base = {a.array: torch.rand(plan.mesh.data[a.array].values.size, generator=g, device="cuda",
                                    dtype=torch.float64) for a in kernel.args}
        out = {}
        for sched in ("stream", "stream-dataflow", "pipelined", "colour"):
            t = {k: v.clone() for k, v in base.items()}
            lp = mp.bind(plan, kernel, tensors=t, schedule=sched)
            for _ in range(2):
                lp.run()
            torch.cuda.synchronize()
            out[sched] = t["res"].cpu().numpy()
        for sched in out:
            assert np.array_equal(out[sched].view(np.uint64), out["colour"].view(np.uint64)), sched
        print("ok")
    """)
    repo = Path(__file__).resolve().parents[1]
    env = dict(__import__("os").environ, MESHPLAN_STREAM_TMA="1", PYTHONPATH=str(repo))
    r = subprocess.run([sys.executable, "-c", code], cwd=repo, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("dims,shape,bs", [((96, 83), "8,8", 128), ((61, 40), "4,6", 48), ((50, 50), "8,8,1", 128)])
def test_quad2d_structured_tiles_extension(dims, shape, bs):
    """Extension: handcrafted bx x by cell tiles for generated quad meshes
    (ragged far edges) -- race-free (checked on execute), widths <= S,
    exact vs the oracle on every schedule, reuse above GPS's."""
    from oracle import loops

    mesh = mp.generate_mesh("quad2d", dims, dtype="f64")
    kernel = mp.kernel_for_mesh("flux", mesh)
    m = mesh.mappings["e2c"]
    want = loops.serial_loop("flux", m.table, mesh.data["q"].view2d(), np.ascontiguousarray(mesh.data["w"].view2d()),
                             _v2(mesh, "res"))
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder=f"structured:{shape}", block_size=bs))
    assert int(np.diff(plan.block_offsets).max()) <= bs
    for sched in SCHEDULES:
        res, _ = mp.execute_hierarchical(plan, kernel, schedule=sched)
        assert bit_equal(_v2(plan.restore_data(res), "res"), want), sched
    gps = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps", block_size=bs))
    assert mp.reuse_factor(plan) > mp.reuse_factor(gps)


def test_quad2d_structured_rejects_3d_shapes():
    mesh = mp.generate_mesh("quad2d", (8, 8), dtype="f64")
    kernel = mp.kernel_for_mesh("flux", mesh)
    with pytest.raises(mp.MeshValidationError):
        mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="structured:2,2,2"))


def test_back_to_back_loops_reading_each_others_increments():
    """Loop B reads (indirectly) the array loop A increments, launched back to
    back on one stream: B must see A's complete result (the streamed
    executor's programmatic-dependent launches never overlap across calls)."""
    mesh = mp.generate_mesh("quad2d", (400, 360), dtype="f64")
    kernel = mp.kernel_for_mesh("flux", mesh)
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps"))
    g = torch.Generator(device="cuda").manual_seed(11)
    n_q = plan.mesh.data["q"].values.size
    n_w = plan.mesh.data["w"].values.size
    X = torch.rand(n_q, generator=g, device="cuda", dtype=torch.float64)
    W = torch.rand(n_w, generator=g, device="cuda", dtype=torch.float64)
    for sched in ("stream", "stream-pull", "stream-dataflow"):
        outs = []
        for sync in (True, False):
            Y = torch.zeros(n_q, device="cuda", dtype=torch.float64)
            Z = torch.zeros(n_q, device="cuda", dtype=torch.float64)
            a = mp.bind(plan, kernel, tensors={"q": X, "w": W, "res": Y}, schedule=sched)
            b = mp.bind(plan, kernel, tensors={"q": Y, "w": W, "res": Z}, schedule=sched)
            for _ in range(3):
                a.run()
                if sync:
                    torch.cuda.synchronize()
                b.run()
                if sync:
                    torch.cuda.synchronize()
            torch.cuda.synchronize()
            outs.append(Z.cpu().numpy())
        assert bit_equal(outs[0], outs[1]), sched


@pytest.mark.parametrize("family,dims,kname", [
    ("quad2d", (1, 1), "flux"), ("quad2d", (1, 2), "flux"), ("quad2d", (2, 1), "flux"), ("quad2d", (3, 3), "flux"),
    ("tri2d", (1, 1), "flux"), ("hex3d-nodes", (1, 1, 1), "scatter8"), ("hex3d-faces", (1, 1, 1), "face-flux"),
    ("hex3d-faces", (2, 1, 1), "face-flux"), ("hex3d-nodes", (2, 3, 1), "scatter8"),
])
def test_tiny_meshes_every_executor(family, dims, kname):
    """Degenerate sizes (no elements, one element, one block smaller than a
    warp): every strategy and schedule equals the oracle."""
    from oracle import loops

    mesh = mp.generate_mesh(family, dims, dtype="f64")
    kernel = mp.kernel_for_mesh(kname, mesh)
    inc = INC_OF[kname]
    m = next(iter(mesh.mappings.values()))
    read = {"flux": "q", "face-flux": "state"}.get(kname)
    direct = {"flux": "w", "scatter8": "stress", "face-flux": "facew"}[kname]
    want = loops.serial_loop(kname, m.table, None if read is None else mesh.data[read].view2d(),
                             np.ascontiguousarray(mesh.data[direct].view2d()), _v2(mesh, inc))
    assert bit_equal(_v2(mp.execute_serial(mesh, kernel), inc), want)
    staging = "increment-only" if kname == "face-flux" else "all-indirect"
    for strategy, reorder in (("global", "none"), ("global", "gps"), ("hier", "none"), ("hier", "gps")):
        cfg = mp.PlanConfig(strategy=strategy, reorder=reorder, staging=staging, block_size=32)
        plan = (mp.build_global_plan if strategy == "global" else mp.build_hierarchical_plan)(mesh, kernel, cfg)
        for sched in (SCHEDULES if strategy == "hier" else ("-",)):
            res, _ = _run(plan, kernel, sched)
            assert bit_equal(_v2(plan.restore_data(res), inc), want), (strategy, reorder, sched)


@pytest.mark.parametrize("bs", [448, 480])
def test_paper_block_sizes_every_schedule(bs):
    """The paper's large blocks: every schedule exact vs
    the oracle (the streamed executor's widest CTA is 480 + 32 threads)."""
    from oracle import loops

    mesh = mp.generate_mesh("quad2d", (120, 110), dtype="f64")
    kernel = mp.kernel_for_mesh("flux", mesh)
    m = mesh.mappings["e2c"]
    want = loops.serial_loop("flux", m.table, mesh.data["q"].view2d(), np.ascontiguousarray(mesh.data["w"].view2d()),
                             _v2(mesh, "res"))
    for reorder in ("none", "gps", "partition"):
        plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder=reorder, block_size=bs))
        for sched in SCHEDULES:
            res, _ = mp.execute_hierarchical(plan, kernel, schedule=sched)
            assert bit_equal(_v2(plan.restore_data(res), "res"), want), (reorder, sched)


@pytest.mark.parametrize("family,dims,kname", [("quad2d", (64, 48), "flux"), ("hex3d-nodes", (10, 9, 8), "scatter8"),
                                               ("hex3d-faces", (9, 8, 7), "face-flux")])
def test_atomic_baseline_exact_on_grid_data(family, dims, kname):
    """Atomics baseline: reassociated sums, exact on the generators' 1/1024
    grid data (every partial sum is representable)."""
    from oracle import loops

    mesh = mp.generate_mesh(family, dims, dtype="f64")
    kernel = mp.kernel_for_mesh(kname, mesh)
    inc = INC_OF[kname]
    m = next(iter(mesh.mappings.values()))
    read = {"flux": "q", "face-flux": "state"}.get(kname)
    direct = {"flux": "w", "scatter8": "stress", "face-flux": "facew"}[kname]
    want = loops.serial_loop(kname, m.table, None if read is None else mesh.data[read].view2d(),
                             np.ascontiguousarray(mesh.data[direct].view2d()), _v2(mesh, inc))
    staging = "increment-only" if kname == "face-flux" else "all-indirect"
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps", staging=staging))
    lp = mp.bind(plan, kernel, schedule="atomic")
    lp.run()
    torch.cuda.synchronize()
    arr = plan.mesh.data[inc]
    res = plan.mesh.with_data(mp.DataArray(arr.name, arr.set, arr.components, lp.tensors[inc].cpu().numpy(), arr.layout))
    assert np.array_equal(_v2(plan.restore_data(res), inc), want)


@pytest.mark.parametrize("kname,family,dims", [("flux", "quad2d", (200, 150)), ("scatter8", "hex3d-nodes", (14, 12, 10)),
                                               ("face-flux", "hex3d-faces", (12, 10, 9))])
def test_block_subsets_cover_the_loop(kname, family, dims):
    """DevicePlan.subset views (the decomposition's core / boundary split):
    running a random split of the blocks as two views equals one full run on
    grid data (each point's increments only change association), every colour
    schedule and executor."""
    mesh = mp.generate_mesh(family, dims, dtype="f64")
    kernel = mp.kernel_for_mesh(kname, mesh)
    staging = "increment-only" if kname == "face-flux" else "all-indirect"
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps", staging=staging, block_size=64))
    inc = INC_OF[kname]
    g = torch.Generator(device="cuda").manual_seed(3)
    mask = torch.rand(plan.num_blocks, generator=g, device="cuda") < 0.6
    for sched in ("stream", "stream-pull", "colour", "pipelined"):
        full = mp.bind(plan, kernel, schedule=sched)
        full.run()
        split = mp.bind(plan, kernel, schedule=sched)
        a, b = plan._device.subset(mask), plan._device.subset(~mask)
        assert a.num_blocks + b.num_blocks == plan.num_blocks
        split.run(sub=a)
        split.run(sub=b)
        torch.cuda.synchronize()
        assert bit_equal(split.tensors[inc].cpu().numpy(), full.tensors[inc].cpu().numpy()), sched
    empty = plan._device.subset(torch.zeros(plan.num_blocks, dtype=torch.bool, device="cuda"))
    assert empty.num_blocks == 0 and empty.launches == 0
    lp = mp.bind(plan, kernel, schedule="stream")
    before = lp.tensors[inc].clone()
    lp.run(sub=empty)
    torch.cuda.synchronize()
    assert torch.equal(lp.tensors[inc], before)
    with pytest.raises(mp.KernelSpecError):
        mp.bind(plan, kernel, schedule="stream-dataflow").run(sub=a)


@pytest.mark.parametrize("family,dims,kname", [("quad2d", (64, 48), "flux"), ("hex3d-nodes", (10, 9, 8), "scatter8"),
                                               ("hex3d-faces", (9, 8, 7), "face-flux"), ("tri2d", (30, 20), "flux")])
def test_temp_array_baseline_is_serial_order(family, dims, kname):
    """Temporary-array baseline (per-(element, slot) temp increments, then a
    per-point fold in element order): bit-identical to the serial loop over
    the plan's numbering for arbitrary (non-grid) data."""
    from oracle import loops

    mesh = mp.generate_mesh(family, dims, dtype="f64")
    rng = np.random.default_rng(5)
    for name, arr in list(mesh.data.items()):
        mesh = mesh.with_data(mp.DataArray(arr.name, arr.set, arr.components,
                                           rng.standard_normal(arr.values.size), arr.layout))
    kernel = mp.kernel_for_mesh(kname, mesh)
    inc = INC_OF[kname]
    staging = "increment-only" if kname == "face-flux" else "all-indirect"
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps", staging=staging))
    pm = plan.mesh
    m = next(iter(pm.mappings.values()))
    read = {"flux": "q", "face-flux": "state"}.get(kname)
    direct = {"flux": "w", "scatter8": "stress", "face-flux": "facew"}[kname]
    want = loops.serial_loop(kname, m.table, None if read is None else pm.data[read].view2d(),
                             np.ascontiguousarray(pm.data[direct].view2d()), _v2(pm, inc))
    lp = mp.bind(plan, kernel, schedule="temp-array")
    assert lp.launches_per_run() == 2
    lp.run()
    torch.cuda.synchronize()
    arr = pm.data[inc]
    got = pm.with_data(mp.DataArray(arr.name, arr.set, arr.components, lp.tensors[inc].cpu().numpy(), arr.layout))
    assert bit_equal(_v2(got, inc), want)


def test_host_stream_steps_equal_single_runs():
    """mp.HostStream: streamed steps over host buffers (H2D, loop, D2H on
    alternating streams) each give the one-step result."""
    mesh = mp.generate_mesh("quad2d", (300, 200), dtype="f64")
    kernel = mp.kernel_for_mesh("flux", mesh)
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps"))
    inputs = {a.array: plan.mesh.data[a.array].values for a in kernel.args}
    ref = mp.bind(plan, kernel, schedule="stream")
    ref.run()
    torch.cuda.synchronize()
    want = ref.tensors["res"].cpu().numpy()
    hs = mp.HostStream(plan, kernel, schedule="stream", depth=2)
    outs = [torch.empty(want.size, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    for k in range(5):
        hs.step(inputs, outs[k % 2])
        if k % 2 == 1:
            hs.synchronize()
            assert all(bit_equal(o.numpy(), want) for o in outs)
    hs.synchronize()
    assert bit_equal(outs[0].numpy(), want)


@pytest.mark.parametrize("kname", ["face-flux", "face-flux-heavy"])
def test_staged_reads_under_increment_only_change_nothing(kname, monkeypatch):
    """Increment-only plans whose read slots are staged slots: the executors
    take the read rows from the staged copy (gpuplan.stage_reads); results
    are bit-identical to reading them from global, every schedule, random
    data."""
    from paper_1802_03749_b200 import gpuplan

    mesh = mp.generate_mesh("hex3d-faces", (10, 9, 8), dtype="f64")
    rng = np.random.default_rng(9)
    for name, arr in list(mesh.data.items()):
        mesh = mesh.with_data(mp.DataArray(arr.name, arr.set, arr.components,
                                           rng.uniform(0.5, 1.5, arr.values.size), arr.layout))
    kernel = mp.kernel_for_mesh(kname, mesh)
    cfg = mp.PlanConfig(reorder="partition", staging="increment-only")
    staged = mp.build_hierarchical_plan(mesh, kernel, cfg)
    assert staged._device.stage_reads
    monkeypatch.setattr(gpuplan, "stage_reads", lambda *a: False)
    direct = mp.build_hierarchical_plan(mesh, kernel, cfg)
    assert not direct._device.stage_reads
    inc = INC_OF[kname]
    for sched in SCHEDULES:
        a, _ = mp.execute_hierarchical(staged, kernel, schedule=sched)
        b, _ = mp.execute_hierarchical(direct, kernel, schedule=sched)
        assert bit_equal(_v2(a, inc), _v2(b, inc)), sched


def test_captured_graph_replays_the_loop():
    """DeviceLoop.capture: a CUDA-graph replay equals a direct execution,
    bit for bit, for the colour schedules (dataflow refuses)."""
    mesh = mp.generate_mesh("quad2d", (200, 160), dtype="f64")
    kernel = mp.kernel_for_mesh("flux", mesh)
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps"))
    for sched in ("stream", "stream-pull", "pipelined", "colour"):
        a = mp.bind(plan, kernel, schedule=sched)
        b = mp.bind(plan, kernel, schedule=sched)
        g = b.capture()  # the warm-up run's increments are undone: capture has no effect
        for _ in range(2):
            a.run()
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        assert bit_equal(a.tensors["res"].cpu().numpy(), b.tensors["res"].cpu().numpy()), sched
    with pytest.raises(mp.KernelSpecError):
        mp.bind(plan, kernel, schedule="stream-dataflow").capture()
    glob = mp.build_global_plan(mesh, kernel, mp.PlanConfig(strategy="global", reorder="gps"))
    a, b = mp.bind(glob, kernel), mp.bind(glob, kernel)
    g = b.capture()
    a.run()
    g.replay()
    torch.cuda.synchronize()
    assert bit_equal(a.tensors["res"].cpu().numpy(), b.tensors["res"].cpu().numpy())


def test_concurrent_threads_with_different_plan_sizes():
    """Threads launching the same executors with different shared-memory sizes
    (different plans) at once: the per-kernel limit only grows, so no launch
    sees a limit lowered by another thread (cudaErrorInvalidValue before)."""
    import threading

    errors = []
    dims = [(60, 40), (90, 70), (40, 30), (120, 50)]

    def worker(d, bs):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                mesh = mp.generate_mesh("quad2d", d, dtype="f64")
                kernel = mp.kernel_for_mesh("flux", mesh)
                plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps", block_size=bs))
                loops = [mp.bind(plan, kernel, schedule=s) for s in ("pipelined", "pipelined-pull", "colour",
                                                                      "stream", "stream-pull")]
                for _ in range(20):
                    for lp in loops:
                        lp.run(torch.cuda.current_stream())
                torch.cuda.current_stream().synchronize()
        except Exception as exc:  # pragma: no cover - surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(d, bs)) for d, bs in zip(dims, (32, 64, 128, 96))]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=300)
    assert not errors, errors


DATAFLOW_SCHEDULES = ("dataflow", "stream-dataflow", "pipelined-dataflow", "pipelined-dataflow-pull")


def test_one_plan_runs_concurrently_on_every_schedule():
    """a finished plan may be executed concurrently.  Loops bound
    to ONE plan on every schedule -- the dataflow ones included, which keep
    per-loop flags and tickets, and whose static-claim grids the library
    chains so two are never co-resident -- run at once from several threads on
    their own streams; every result equals the single-run colour schedule bit
    for bit (random data: any ordering slip shows).  One dataflow loop driven
    from two streams alternately is ordered by its own event chain."""
    import threading

    mesh = mp.generate_mesh("quad2d", (160, 150), dtype="f64")
    rng = np.random.default_rng(5)
    mesh = mesh.with_data(*[mp.DataArray(a.name, a.set, a.components, rng.standard_normal(a.values.size), a.layout)
                            for a in mesh.data.values()])
    kernel = mp.kernel_for_mesh("flux", mesh)
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps", block_size=64))
    reps = 6
    ref = mp.bind(plan, kernel, schedule="colour")
    for _ in range(reps):
        ref.run()
    torch.cuda.synchronize()
    want = ref.tensors["res"].cpu().numpy()
    errors, results = [], {}

    def worker(sched, k):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                lp = mp.bind(plan, kernel, schedule=sched)
                for _ in range(reps):
                    lp.run(torch.cuda.current_stream())
                torch.cuda.current_stream().synchronize()
                results[(sched, k)] = lp.tensors["res"].cpu().numpy()
        except Exception as exc:  # pragma: no cover - surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(s, k)) for k in range(2)
               for s in DATAFLOW_SCHEDULES + ("stream", "colour", "pipelined-pull")]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=300)
    assert not errors, errors
    assert len(results) == len(threads)
    for key, got in results.items():
        assert bit_equal(got, want), key
    # one dataflow loop, executions alternating between two streams
    for sched in DATAFLOW_SCHEDULES:
        lp = mp.bind(plan, kernel, schedule=sched)
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        for i in range(reps):
            lp.run(streams[i % 2])
        torch.cuda.synchronize()
        assert bit_equal(lp.tensors["res"].cpu().numpy(), want), sched


def test_host_stream_on_a_dataflow_schedule():
    """mp.HostStream with depth 2 on the dataflow schedules: each step's
    loop has its own flags and tickets, so steps in flight together are
    exact (they used to share the plan's)."""
    mesh = mp.generate_mesh("quad2d", (220, 130), dtype="f64")
    kernel = mp.kernel_for_mesh("flux", mesh)
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps"))
    inputs = {a.array: plan.mesh.data[a.array].values for a in kernel.args}
    ref = mp.bind(plan, kernel, schedule="stream")
    ref.run()
    torch.cuda.synchronize()
    want = ref.tensors["res"].cpu().numpy()
    for sched in DATAFLOW_SCHEDULES:
        hs = mp.HostStream(plan, kernel, schedule=sched, depth=2)
        outs = [torch.empty(want.size, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        for k in range(6):
            hs.step(inputs, outs[k % 2])
            if k % 2 == 1:
                hs.synchronize()
                assert all(bit_equal(o.numpy(), want) for o in outs), sched

"""The gather-form executor (``schedule="gather"``, exec_hier_gather.cu).

Lanes own (element, slot) refs instead of elements and each staged row's
refs are summed in thread-colour order by a shuffle chain, so its results
must be the reference executor's bit for bit (simulator.py:525-656: zeroed
shared row, per-colour adds, one write-back) -- checked on the reference's
own plans with non-quantised random data, and against the streamed push
executor on larger meshes of every family and block layout (GPS strips,
k-way partitions, quad tiles, structured hex blocks, 448/480-element
blocks), back to back, through block subsets and as a CUDA graph.
"""

import numpy as np
import pytest
import torch

import paper_1802_03749_b200 as mp
from conftest import INC_OF, bit_equal, case_mesh, golden_cases, load_case
from helpers import reference_plan

pytestmark = pytest.mark.gpu

CASES = [c for c in golden_cases() if c["strategy"] == "hier" and c["layout"] == "aos"]


def _ids(c):
    return f"{c['file']}-{c['family']}-{c['kernel']}-{c['dtype']}-{c['reorder']}"


@pytest.mark.parametrize("rec", CASES, ids=_ids)
def test_gather_on_reference_plan_bit_exact(rec):
    z = load_case(rec)
    rmesh = case_mesh(rec, random=True, arrays=z)
    kernel = mp.kernel_for_mesh(rec["kernel"], rmesh)
    plan = reference_plan(rec, z, rmesh, kernel)
    res, rep = mp.execute_hierarchical(plan, kernel, schedule="gather")
    assert bit_equal(np.ascontiguousarray(res.data[INC_OF[rec["kernel"]]].view2d()), z["rand_exec_inc"])
    assert rep.schedule == "gather"


MESHES = [("quad2d", (300, 260), "flux", "gps", 128), ("quad2d", (300, 260), "flux", "structured:8,8", 128),
          ("quad2d", (300, 260), "flux", "structured:16,16", 480), ("quad2d", (120, 100), "flux", "partition", 128),
          ("tri2d", (200, 180), "flux", "gps", 128), ("tri2d", (200, 180), "flux-noread", "none", 96),
          ("hex3d-nodes", (24, 20, 18), "scatter8", "none", 128),
          ("hex3d-nodes", (24, 20, 16), "scatter8", "structured:4,4,8", 128),
          ("hex3d-faces", (24, 20, 18), "face-flux", "none", 128),
          ("hex3d-faces", (16, 16, 16), "face-flux", "structured:4,4,8", 480),
          ("hex3d-faces", (20, 18, 16), "face-flux-heavy", "partition", 256)]


@pytest.mark.parametrize("family,dims,kname,reorder,bs", MESHES,
                         ids=[f"{m[0]}-{m[2]}-{m[3]}-{m[4]}" for m in MESHES])
def test_gather_equals_push_on_random_data(family, dims, kname, reorder, bs):
    mesh = mp.generate_mesh(family, dims, dtype="f64")
    kernel = mp.kernel_for_mesh(kname, mesh)
    staging = "increment-only" if kname.startswith("face-flux") else "all-indirect"
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder=reorder, block_size=bs, staging=staging))
    g = torch.Generator(device="cuda").manual_seed(11)
    base = {}
    for a in kernel.args:
        if a.array not in base:
            n = plan.mesh.data[a.array].values.size
            base[a.array] = torch.rand(n, generator=g, device="cuda", dtype=torch.float64) * 2 - 1
    inc = INC_OF[kname]
    out = {}
    for sched in ("stream", "colour", "gather"):
        t = {k: v.clone() for k, v in base.items()}
        lp = mp.bind(plan, kernel, tensors=t, schedule=sched)
        for _ in range(3):  # back to back: the next execution reads this one's increments
            lp.run()
        torch.cuda.synchronize()
        out[sched] = t[inc].cpu().numpy()
    assert bit_equal(out["gather"], out["colour"])
    assert bit_equal(out["gather"], out["stream"])


def test_gather_subsets_and_graph_replay():
    """Core / boundary block views run one after the other equal one full
    execution; a captured execution replays to the same bits."""
    mesh = mp.generate_mesh("quad2d", (160, 140), dtype="f64")
    kernel = mp.kernel_for_mesh("flux", mesh)
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="structured:8,8"))
    g = torch.Generator(device="cuda").manual_seed(5)
    base = {a.array: torch.rand(plan.mesh.data[a.array].values.size, generator=g, device="cuda",
                                dtype=torch.float64) for a in kernel.args}
    full = {k: v.clone() for k, v in base.items()}
    mp.bind(plan, kernel, tensors=full, schedule="gather").run()
    split = {k: v.clone() for k, v in base.items()}
    lp = mp.bind(plan, kernel, tensors=split, schedule="gather")
    mask = torch.arange(plan.num_blocks, device="cuda") % 3 == 0
    lp.run(sub=plan._device.subset(mask))
    lp.run(sub=plan._device.subset(~mask))
    graphed = {k: v.clone() for k, v in base.items()}
    lg = mp.bind(plan, kernel, tensors=graphed, schedule="gather")
    gr = lg.capture()
    gr.replay()
    torch.cuda.synchronize()
    # the split runs every block once; points shared by the two views get the
    # first view's blocks first (reassociation only)
    assert bit_equal(graphed["res"].cpu().numpy(), full["res"].cpu().numpy())
    assert np.allclose(split["res"].cpu().numpy(), full["res"].cpu().numpy(), rtol=1e-12, atol=1e-12)


def test_gather_refuses_soa_plans():
    mesh = mp.generate_mesh("quad2d", (40, 30), dtype="f64")
    kernel = mp.kernel_for_mesh("flux", mesh)
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps", layout="soa"))
    with pytest.raises(mp.KernelSpecError):
        mp.execute_hierarchical(plan, kernel, schedule="gather")

"""Generate golden fixtures from the REAL reference package (run in the build
container, where /root/reference exists; the GPU box never runs this).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

For each case it stores the reference plan arrays (permutations, colours,
offsets, staging lists), the reference ``execute_serial`` result on the
generator's quantised data, and -- for bit-exact same-plan parity -- the
reference ``execute_global`` / ``execute_hierarchical`` and ``execute_serial``
results on NON-quantised random data (stored with the fixture, so the check
does not depend on the RNG stream of whatever numpy the GPU box has).
Reference versions at generation time: numpy 2.3.5, numba 0.65.0.
"""

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import meshplan as mp  # noqa: E402
from meshplan.bench_kernels import generate_mesh, kernel_for_mesh  # noqa: E402
from meshplan.mesh import DataArray  # noqa: E402

OUT = Path(__file__).resolve().parent

# (family, dims, kernel, dtype, staging)
MESHES = [
    ("quad2d", (16, 16), "flux", "f64", "all-indirect"),
    ("quad2d", (12, 9), "flux-noread", "f32", "all-indirect"),
    ("quad2d", (10, 10), "face-flux", "i64", "increment-only"),
    ("tri2d", (10, 10), "flux", "f32", "all-indirect"),
    ("tri2d", (8, 7), "flux", "i32", "all-indirect"),
    ("hex3d-nodes", (6, 6, 8), "scatter8", "f64", "all-indirect"),
    ("hex3d-nodes", (4, 4, 4), "scatter8", "i64", "all-indirect"),
    ("hex3d-faces", (5, 5, 6), "face-flux", "f64", "increment-only"),
    ("hex3d-faces", (4, 4, 5), "face-flux-heavy", "f64", "all-indirect"),
    ("hex3d-faces", (4, 4, 4), "face-flux-heavy", "f32", "all-indirect"),
]
STRATEGIES = [("global", "none"), ("global", "gps"), ("global", "partition"),
              ("hier", "none"), ("hier", "gps"), ("hier", "partition")]
STRUCTURED = {"hex3d-nodes": "structured:2,2,4", "hex3d-faces": None}


def randomise(mesh, seed):
    """Same mesh, non-quantised values (float) / wider ints, zero increments kept."""
    rng = np.random.default_rng(1000 + seed)
    arrays = []
    for name, a in mesh.data.items():
        v = a.values
        if name in ("res", "force", "flux"):
            if v.dtype.kind == "f":
                v = rng.standard_normal(v.size).astype(v.dtype)  # non-zero initial increments too
            else:
                v = rng.integers(-50, 50, v.size).astype(v.dtype)
        elif v.dtype.kind == "f":
            v = rng.standard_normal(v.size).astype(v.dtype)
        else:
            v = rng.integers(-1000, 1000, v.size).astype(v.dtype)
        arrays.append(DataArray(a.name, a.set, a.components, v, a.layout))
    return mesh.with_data(*arrays)


def inc_name(kname):
    return {"flux": "res", "flux-noread": "res", "scatter8": "force"}.get(kname, "flux")


def main():
    manifest = []
    idx = 0
    for mi, (family, dims, kname, dtype, staging) in enumerate(MESHES):
        mesh = generate_mesh(family, dims, seed=mi, dtype=dtype)
        kernel = kernel_for_mesh(kname, mesh)
        rmesh = randomise(mesh, mi)
        inc = inc_name(kname)
        serial = mp.execute_serial(mesh, kernel).data[inc].view2d()
        serial_r = mp.execute_serial(rmesh, kernel).data[inc].view2d()
        strategies = list(STRATEGIES)
        if STRUCTURED.get(family):
            strategies.append(("hier", STRUCTURED[family]))
        for si, (strategy, reorder) in enumerate(strategies):
            layout = "aos" if (mi + si) % 2 == 0 else "soa"
            bs = (64, 128, 96, 50)[(mi + si) % 4]
            cfg = mp.PlanConfig(strategy=strategy, reorder=reorder, layout=layout, staging=staging, block_size=bs)
            build = mp.build_global_plan if strategy == "global" else mp.build_hierarchical_plan
            plan = build(mesh, kernel, cfg)
            rplan = build(rmesh, kernel, cfg)
            run = mp.execute_global if strategy == "global" else mp.execute_hierarchical
            res, _ = run(plan, kernel)
            res_r, _ = run(rplan, kernel)
            m = next(iter(mesh.mappings.values()))
            rec = {
                "family": family, "dims": list(dims), "kernel": kname, "dtype": dtype, "seed": mi,
                "strategy": strategy, "reorder": reorder, "layout": layout, "staging": staging, "block_size": bs,
            }
            arrs = {
                "elem_fwd": plan.set_perms[m.from_set.name].forward,
                "point_fwd": plan.set_perms[m.to_set.name].forward,
                "plan_table": plan.mesh.mappings[m.name].table,
                "serial_inc": serial,
                "rand_serial_inc": serial_r,
                "rand_exec_inc": res_r.data[inc].view2d(),
                "exec_inc": res.data[inc].view2d(),
            }
            for name, a in rmesh.data.items():  # random inputs, original numbering, (rows, comps)
                arrs[f"rand_{name}"] = np.ascontiguousarray(a.view2d())
            if strategy == "global":
                arrs["colours"] = plan.colours.colours
                arrs["colour_offsets"] = plan.colour_offsets
                rec["num_colours"] = plan.num_colours
            else:
                arrs["block_offsets"] = plan.block_offsets
                arrs["block_colours"] = plan.block_colours.colours
                arrs["thread_colours"] = plan.thread_colours
                arrs["thread_colour_counts"] = plan.thread_colour_counts
                ((sk, (sp, sids)),) = plan.staged.items()
                ((wk, (wp, wids)),) = plan.written.items()
                arrs.update(staged_ptr=sp, staged_ids=sids, written_ptr=wp, written_ids=wids,
                            shared_bytes=plan.shared_bytes)
                rec["num_block_colours"] = plan.block_colours.num_colours
                rec["refs_per_element"] = plan.refs_per_element
                rec["reuse_factor"] = mp.reuse_factor(plan)
                rec["partition_meta"] = {k: (float(v) if isinstance(v, float) else v)
                                         for k, v in plan.partition_meta.items()}
            fname = f"case{idx:03d}.npz"
            np.savez_compressed(OUT / fname, **arrs)
            rec["file"] = fname
            manifest.append(rec)
            idx += 1
            print(fname, family, dims, kname, dtype, strategy, reorder, layout, bs, flush=True)
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1, default=lambda o: o.tolist()) + "\n")


if __name__ == "__main__":
    main()

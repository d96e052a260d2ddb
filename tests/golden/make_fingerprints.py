"""Freeze fingerprints of the REAL reference's plans and loop results at the
BASELINE config sizes (run in the build container, where /root/reference
exists; the GPU box only reads the committed ``fingerprints.json``).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_fingerprints.py [C1 C2 ...]

The configs are SURVEY.md 8(d)'s (all ``seed=0``, reference generators):
C1 quad2d 848^2 flux f64, C2 tri2d 1095^2 flux f32, C3 hex3d-nodes 160^3
scatter8 f64, C4 hex3d-faces 200^3 face-flux f64 (and the 60^3 stand-in
SURVEY 6 uses for plans), C5 quad2d 5657^2 flux f64.  Full arrays at these
sizes are hundreds of MB, so each array is stored as a CRC32 of its bytes
(int arrays as little-endian int64, float arrays as their own dtype) plus
its length: the GPU tests recompute the same CRC over the device result.

Recorded per config: the reference ``execute_serial`` result (simulator.py:
215-242) on the generator's quantised data, and for each planned
(strategy, reorder) the plan arrays (plan.py:408-579) -- and, where the
reference simulator finishes in seconds (C1), its ``execute_global`` /
``execute_hierarchical`` result on non-quantised random data (the
same-plan bit-exact check; the random values come from
``np.random.default_rng(7)`` in the test too).
Reference versions at generation time: numpy 2.3.5, numba 0.65.0.
"""

import json
import sys
import time
import zlib
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import meshplan as mp  # noqa: E402
from meshplan.bench_kernels import generate_mesh, kernel_for_mesh  # noqa: E402
from meshplan.mesh import DataArray  # noqa: E402

OUT = Path(__file__).resolve().parent / "fingerprints.json"

# name: (family, dims, kernel, dtype, staging, [(strategy, reorder)], random-data executor strategies)
CONFIGS = {
    "C1": ("quad2d", (848, 848), "flux", "f64", "all-indirect",
           [("global", "none"), ("global", "gps"), ("global", "partition"),
            ("hier", "none"), ("hier", "gps"), ("hier", "partition")],
           [("global", "gps"), ("hier", "gps"), ("hier", "partition")]),
    "C2": ("tri2d", (1095, 1095), "flux", "f32", "all-indirect",
           [("global", "none"), ("hier", "none"), ("hier", "gps"), ("hier", "partition")], []),
    "C3": ("hex3d-nodes", (160, 160, 160), "scatter8", "f64", "all-indirect",
           [("global", "none"), ("hier", "none"), ("hier", "gps")], []),
    "C4s": ("hex3d-faces", (60, 60, 60), "face-flux", "f64", "increment-only",
            [("hier", "none"), ("hier", "partition")], [("hier", "partition")]),
    "C4": ("hex3d-faces", (200, 200, 200), "face-flux", "f64", "increment-only", [("hier", "partition")], []),
    # the bench's C4 headline plan: the same k-way partition at block size 256
    "C4k256": ("hex3d-faces", (200, 200, 200), "face-flux", "f64", "increment-only", [("hier", "partition")], [],
               256),
    "C5": ("quad2d", (5657, 5657), "flux", "f64", "all-indirect", [("hier", "gps"), ("global", "gps")], []),
}
INC = {"flux": "res", "flux-noread": "res", "scatter8": "force", "face-flux": "flux", "face-flux-heavy": "flux"}


def crc(a) -> dict:
    a = np.ascontiguousarray(a)
    if a.dtype.kind in "iu":
        a = a.astype("<i8")
    return {"crc32": zlib.crc32(a.tobytes()) & 0xFFFFFFFF, "len": int(a.size)}


def randomise(mesh, inc):
    """Non-quantised inputs (and non-zero initial increments), rng seed 7,
    arrays in mesh.data order (the test draws them the same way)."""
    rng = np.random.default_rng(7)
    arrays = []
    for name, a in mesh.data.items():
        v = rng.standard_normal(a.values.size).astype(a.values.dtype)
        arrays.append(DataArray(a.name, a.set, a.components, v, a.layout))
    return mesh.with_data(*arrays)


def plan_record(plan, m):
    rec = {"elem_fwd": crc(plan.set_perms[m.from_set.name].forward),
           "point_fwd": crc(plan.set_perms[m.to_set.name].forward)}
    if isinstance(plan, mp.GlobalPlan):
        rec["colours"] = crc(plan.colours.colours)
        rec["colour_offsets"] = [int(x) for x in plan.colour_offsets]
        rec["num_colours"] = int(plan.num_colours)
    else:
        ((_, (sp, sids)),) = plan.staged.items()
        ((_, (wp, wids)),) = plan.written.items()
        rec.update(block_offsets=crc(plan.block_offsets), block_colours=crc(plan.block_colours.colours),
                   num_block_colours=int(plan.block_colours.num_colours),
                   block_colour_counts=[int(x) for x in plan.block_colours.counts],
                   thread_colours=crc(plan.thread_colours), thread_colour_counts=crc(plan.thread_colour_counts),
                   staged_ptr=crc(sp), staged_ids=crc(sids), written_ptr=crc(wp), written_ids=crc(wids),
                   shared_bytes=crc(plan.shared_bytes), num_blocks=int(len(plan.block_offsets) - 1),
                   reuse_factor=float(mp.reuse_factor(plan)),
                   partition_meta={k: (float(v) if isinstance(v, (float, np.floating)) else
                                       (int(v) if isinstance(v, (int, np.integer, bool)) else v))
                                   for k, v in plan.partition_meta.items()})
    return rec


def main(names):
    out = json.loads(OUT.read_text()) if OUT.exists() else {}
    for name in names:
        family, dims, kname, dtype, staging, strategies, rand_runs = CONFIGS[name][:7]
        bs = CONFIGS[name][7] if len(CONFIGS[name]) > 7 else 128
        t0 = time.time()
        mesh = generate_mesh(family, dims, seed=0, dtype=dtype)
        kernel = kernel_for_mesh(kname, mesh)
        inc = INC[kname]
        m = next(iter(mesh.mappings.values()))
        rec = {"family": family, "dims": list(dims), "kernel": kname, "dtype": dtype, "staging": staging,
               "seed": 0, "block_size": bs, "layout": "aos", "n_elements": int(m.from_set.size),
               "n_points": int(m.to_set.size)}
        serial = mp.execute_serial(mesh, kernel).data[inc].view2d()
        rec["serial"] = crc(serial)
        rec["serial_abs_sum"] = float(np.abs(serial).sum())
        print(name, "serial", round(time.time() - t0, 1), "s", flush=True)
        rmesh = randomise(mesh, inc) if rand_runs else None
        if rand_runs:
            rec["rand_serial"] = crc(mp.execute_serial(rmesh, kernel).data[inc].view2d())
        plans = {}
        for strategy, reorder in strategies:
            t1 = time.time()
            cfg = mp.PlanConfig(strategy=strategy, reorder=reorder, layout="aos", staging=staging, block_size=bs)
            build = mp.build_global_plan if strategy == "global" else mp.build_hierarchical_plan
            src = rmesh if (strategy, reorder) in rand_runs else mesh
            plan = build(src, kernel, cfg)
            prec = plan_record(plan, m)
            prec["build_s"] = round(time.time() - t1, 1)
            if (strategy, reorder) in rand_runs:
                t2 = time.time()
                run = mp.execute_global if strategy == "global" else mp.execute_hierarchical
                res, _ = run(plan, kernel)
                prec["rand_exec"] = crc(plan.restore_data(res).data[inc].view2d())
                prec["rand_exec_s"] = round(time.time() - t2, 1)
            plans[f"{strategy}/{reorder}"] = prec
            print(name, strategy, reorder, prec["build_s"], "s", flush=True)
            out.setdefault(name, {}).update(rec)
            out[name].setdefault("plans", {}).update(plans)
            OUT.write_text(json.dumps(out, indent=1) + "\n")
        out.setdefault(name, {}).update(rec)
        out[name].setdefault("plans", {}).update(plans)
        OUT.write_text(json.dumps(out, indent=1) + "\n")
        print(name, "done", round(time.time() - t0, 1), "s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CONFIGS))

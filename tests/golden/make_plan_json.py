"""Plan files written by the REAL reference (``meshplan.save_plan``,
plan.py:679-685, JSON with the mesh fingerprint), frozen as fixtures for the
interoperability tests (tests/test_plan_interop.py).  Run in the build
container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_plan_json.py
"""

import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import meshplan as mp  # noqa: E402
from meshplan.bench_kernels import generate_mesh, kernel_for_mesh  # noqa: E402

OUT = Path(__file__).resolve().parent / "plans"
# name: family, dims, kernel, dtype, PlanConfig kwargs
CASES = {
    "quad2d_flux_hier_gps": ("quad2d", (14, 11), "flux", "f64", dict(strategy="hier", reorder="gps", block_size=32)),
    "quad2d_flux_global_none": ("quad2d", (9, 7), "flux", "f64", dict(strategy="global", reorder="none")),
    "tri2d_flux_hier_partition": ("tri2d", (9, 8), "flux", "f32",
                                  dict(strategy="hier", reorder="partition", block_size=24, layout="soa")),
    "hex3d_faces_hier_structured": ("hex3d-faces", (4, 4, 4), "face-flux", "f64",
                                    dict(strategy="hier", reorder="structured:2,2,2", block_size=64,
                                         staging="increment-only")),
    "hex3d_nodes_global_gps": ("hex3d-nodes", (4, 3, 3), "scatter8", "i64", dict(strategy="global", reorder="gps")),
}


def main():
    OUT.mkdir(exist_ok=True)
    manifest = {}
    for name, (family, dims, kname, dtype, kw) in CASES.items():
        mesh = generate_mesh(family, dims, seed=0, dtype=dtype)
        kernel = kernel_for_mesh(kname, mesh)
        cfg = mp.PlanConfig(**kw)
        build = mp.build_global_plan if cfg.strategy == "global" else mp.build_hierarchical_plan
        plan = build(mesh, kernel, cfg)
        path = OUT / f"{name}.json"
        mp.save_plan(plan, path, mesh=mesh)
        manifest[name] = {"family": family, "dims": list(dims), "kernel": kname, "dtype": dtype, "config": kw}
        print(name, path.stat().st_size, "bytes")
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()

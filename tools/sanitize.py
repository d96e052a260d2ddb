"""Small loops through every executor / schedule, for compute-sanitizer."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1802_03749_b200 as mp  # noqa: E402

cases = [("quad2d", (40, 30), "flux", "all-indirect"), ("hex3d-nodes", (6, 5, 4), "scatter8", "all-indirect"),
         ("hex3d-faces", (6, 5, 4), "face-flux", "increment-only"), ("tri2d", (20, 16), "flux", "all-indirect")]
scheds = sys.argv[1].split(",") if len(sys.argv) > 1 else ["stream", "stream-pull", "stream-dataflow", "pipelined",
                                                           "pipelined-pull", "colour", "dataflow", "atomic",
                                                           "temp-array"]
for fam, dims, kname, staging in cases:
    mesh = mp.generate_mesh(fam, dims, dtype="f64")
    kernel = mp.kernel_for_mesh(kname, mesh)
    for reorder in ("none", "gps"):
        plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder=reorder, staging=staging, block_size=32))
        for sc in scheds:
            lp = mp.bind(plan, kernel, schedule=sc)
            lp.run()
            lp.run()
        g = mp.build_global_plan(mesh, kernel, mp.PlanConfig(strategy="global", reorder=reorder))
        mp.bind(g, kernel).run()
torch.cuda.synchronize()
print("sanitize run ok")

"""Direct launches vs a captured CUDA graph of one loop execution."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import statistics  # noqa: E402

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1802_03749_b200 as mp  # noqa: E402

for cfg_name in sys.argv[1:] or ["C1", "C2"]:
    mesh, kernel, staging = bench.make_mesh(cfg_name)
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="gps", staging=staging))
    lp = mp.bind(plan, kernel, schedule="stream")
    flush = bench.L2Flusher(True)
    direct = bench.time_steps(lp.run, 50, 5, flush)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        lp.run(s)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        lp.run(torch.cuda.current_stream())
    graphed = bench.time_steps(g.replay, 50, 5, flush)
    nf = bench.L2Flusher(False)
    d2 = bench.time_steps(lp.run, 50, 5, nf)
    g2 = bench.time_steps(g.replay, 50, 5, nf)
    print(f"{cfg_name}: direct {statistics.median(direct):.4f} ms, graph {statistics.median(graphed):.4f} ms "
          f"(no flush: {statistics.median(d2):.4f} / {statistics.median(g2):.4f})", flush=True)

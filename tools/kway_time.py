import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1802_03749_b200 as mp
fam, dims = sys.argv[1], tuple(int(x) for x in sys.argv[2].split(","))
kname = sys.argv[3]
mesh = mp.generate_mesh(fam, dims, dtype="f64")
kernel = mp.kernel_for_mesh(kname, mesh)
t = time.perf_counter()
plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder="partition", staging="increment-only" if "face" in kname else "all-indirect"))
print("total", time.perf_counter() - t, getattr(plan, "_timings", ""))

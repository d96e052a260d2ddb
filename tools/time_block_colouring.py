"""Block colouring at the BASELINE configs: the GPU pass (mp_plan_block_colours)
vs the native host C++ greedy (mp_greedy_colour_csr) on the same written lists,
results compared.  python tools/time_block_colouring.py [C1 C3 C4 C5]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1802_03749_b200 import gpuplan  # noqa: E402
from paper_1802_03749_b200.colouring import colour_csr_least_loaded  # noqa: E402

REORDER = {"C1": "gps", "C2": "gps", "C3": "none", "C4": "none", "C5": "gps"}
for cfg in sys.argv[1:] or ["C1", "C2", "C3", "C5"]:
    import paper_1802_03749_b200 as mp

    mesh, kernel, staging = bench.make_mesh(cfg)
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder=REORDER[cfg], staging=staging))
    ((_, (wp, wi)),) = plan.written.items()
    off = torch.as_tensor(wp.astype(np.int32), device="cuda")
    ids = torch.as_tensor(wi.astype(np.int32), device="cuda")
    gpuplan.colour_blocks_device(off, ids)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    col, num, _ = gpuplan.colour_blocks_device(off, ids)
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref = colour_csr_least_loaded(wp, wi, int(wi.max()) + 1)
    t_host = time.perf_counter() - t0
    same = np.array_equal(col.cpu().numpy(), ref.colours) and np.array_equal(plan.block_colours.colours, ref.colours)
    print(f"{cfg}: {len(wp) - 1} blocks, {num} colours, {len(wi)} written refs: GPU {t_gpu * 1e3:.1f} ms, "
          f"host C++ {t_host * 1e3:.1f} ms, identical={same}", flush=True)

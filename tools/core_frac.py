"""Core / boundary block split of one rank's local plan (C5 or C1 slabs)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1802_03749_b200 as mp
from paper_1802_03749_b200 import decomp
from paper_1802_03749_b200.workloads import quad2d_table

nx = ny = int(sys.argv[1]) if len(sys.argv) > 1 else 5657
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
reorder = sys.argv[3] if len(sys.argv) > 3 else "gps"
bounds, xs = decomp.slab_bounds(nx, ny, world)
for r in (0, world // 2):
    t, g = quad2d_table(nx, ny, int(xs[r]), int(xs[r + 1]))
    halos = []
    for rr in range(world):
        if rr == r:
            pts = np.unique(t)
            halos.append(pts[(pts < bounds[r]) | (pts >= bounds[r + 1])])
        else:
            halos.append(np.zeros(0, dtype=np.int64))
    # other ranks' halos only matter for export rows; this rank's own split is what we measure
    dec = decomp.decompose(t, g, bounds, r, world, lambda obj: halos)
    mesh = decomp.local_flux_mesh(t, g, dec, np.zeros((dec.n_local, 4)), np.zeros((len(g), 2)),
                                  np.zeros((dec.n_local, 4)))
    kernel = mp.kernel_for_mesh("flux", mesh)
    dl = decomp.DistributedLoop(mesh, kernel, dec, decomp.ThreadTransport(decomp.ThreadHub(), r),
                                mp.PlanConfig(reorder=reorder, block_size=128), "stream")
    core = dl.core_blocks()
    print(f"rank {r}/{world} {reorder}: {int(core.sum())} core of {core.numel()} blocks "
          f"({float(core.float().mean()):.4f}); halo points {dec.n_local - dec.n_owned}; "
          f"launches core {dl.core.launches} boundary {dl.boundary.launches}", flush=True)

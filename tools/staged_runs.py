"""Runs of consecutive ids in each block's staged list (how compressible the
staged-id lists are), per config and block layout."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1802_03749_b200 as mp  # noqa: E402

for cfg, reorder, bs in (("C1", "gps", 128), ("C2", "gps", 128), ("C3", "none", 128), ("C5", "gps", 128),
                         ("C4", "partition", 256)):
    mesh, kernel, staging = bench.make_mesh(cfg)
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder=reorder, staging=staging, block_size=bs))
    d = plan._device
    meta = d.meta.long()
    s0, ns = meta[:, 2], meta[:, 3]
    nb = ns.numel()
    dev = s0.device
    blk = torch.repeat_interleave(torch.arange(nb, device=dev), ns)
    first = torch.cumsum(ns, 0) - ns
    ids = d.staged_ids.long()[s0[blk] + torch.arange(blk.numel(), device=dev) - first[blk]]
    start = torch.ones_like(ids, dtype=torch.bool)
    start[1:] = (ids[1:] != ids[:-1] + 1) | (blk[1:] != blk[:-1])
    runs = torch.bincount(blk[start], minlength=nb)
    h = torch.bincount(runs.clamp(max=8)).cpu().tolist()
    print(f"{cfg} {reorder} bs{bs}: blocks {nb} staged {ids.numel()} runs/block mean {runs.float().mean():.2f} "
          f"hist(0..8+) {h} <=2: {(runs <= 2).float().mean():.3f} <=3: {(runs <= 3).float().mean():.3f}", flush=True)
    del plan, d, mesh
    torch.cuda.empty_cache()

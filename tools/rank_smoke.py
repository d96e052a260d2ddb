"""Run bench.py's multi-GPU rank path (decomp.bench_rank: NCCL, halo exchange,
core/boundary overlap) with the world size torchrun gives, including 1 --
a smoke test of that path on a single-GPU box:
  torchrun --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 tools/rank_smoke.py --config C1
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1802_03749_b200 import decomp  # noqa: E402

import argparse  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gpus", type=int, default=1)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--config", default="C1")
ap.add_argument("--reorder", default=None)
ap.add_argument("--block-size", type=int, default=128)
ap.add_argument("--schedule", default="best")
ap.add_argument("--cpu-seconds", type=float, default=0.0)
ap.add_argument("--transport", default="peer", choices=("peer", "nccl"))
args, _ = ap.parse_known_args()
if args.reorder is None:
    args.reorder = bench.DEFAULT_REORDER[args.config]
sys.exit(decomp.bench_rank(args, int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))))

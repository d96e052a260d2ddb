"""Profiling driver: build one plan, then run the loop a few times (for ncu).

    python tools/prof_loop.py --config C5 --strategy hier --schedule colour --runs 3
"""

import argparse
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--strategy", default="hier", choices=("hier", "global"))
    ap.add_argument("--schedule", default="colour")
    ap.add_argument("--reorder", default="gps")
    ap.add_argument("--layout", default="aos")
    ap.add_argument("--block-size", type=int, default=128)
    ap.add_argument("--runs", type=int, default=3)
    ap.add_argument("--timed", type=int, default=1)
    ap.add_argument("--lags", default="")
    ap.add_argument("--staging", default=None, help="override the config's staging")
    args = ap.parse_args()

    import torch

    import bench
    import paper_1802_03749_b200 as mp

    mesh, kernel, staging = bench.make_mesh(args.config)
    staging = args.staging or staging
    cfg = mp.PlanConfig(strategy=args.strategy, reorder=args.reorder, layout=args.layout, staging=staging,
                        block_size=args.block_size)
    t0 = time.perf_counter()
    plan = (mp.build_global_plan if args.strategy == "global" else mp.build_hierarchical_plan)(mesh, kernel, cfg)
    print(f"plan {time.perf_counter() - t0:.2f}s {getattr(plan, '_timings', '')}", flush=True)
    if args.strategy == "hier":
        print(f"blocks {plan.num_blocks} block colours {plan.block_colours.num_colours} "
              f"reuse {mp.reuse_factor(plan):.3f} thread colours mean {plan.thread_colour_counts.mean():.2f}",
              flush=True)
    ub = mp.useful_bytes(kernel, mesh)
    scheds = args.schedule.split(",")
    lags = [int(x) for x in args.lags.split(",")] if args.lags else [None]
    for sched in scheds:
        for lag in (lags if "dataflow" in sched else [None]):
            if lag is not None:
                plan._device.reschedule(lag)
            loop = mp.bind(plan, kernel, schedule=sched)
            torch.cuda.synchronize()
            for _ in range(args.runs):
                loop.run()
            torch.cuda.synchronize()
            ts = []
            for _ in range(args.timed):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                loop.run()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = sorted(ts)[len(ts) // 2]
            print(f"{args.strategy}/{sched} lag={lag}: {ms:.4f} ms  {ub / ms / 1e6:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()

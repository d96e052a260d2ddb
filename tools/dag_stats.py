"""Dataflow-order diagnostics: ticket distance from each block to its nearest
predecessor (how far ahead a predecessor finishes), per lag.

    python tools/dag_stats.py --config C5 --lags 2048,4096,8192
"""
import argparse
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--reorder", default="gps")
    ap.add_argument("--lags", default="2048,4096,8192")
    args = ap.parse_args()
    import torch

    import bench
    import paper_1802_03749_b200 as mp

    mesh, kernel, staging = bench.make_mesh(args.config)
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder=args.reorder, staging=staging))
    mp.bind(plan, kernel, schedule="stream-dataflow")
    dp = plan._device
    for lag in [int(x) for x in args.lags.split(",")]:
        dp.reschedule(lag)
        nb = dp.order.numel()
        tick = torch.empty(nb, dtype=torch.long, device="cuda")
        tick[dp.order.long()] = torch.arange(nb, device="cuda")
        po = dp.pred_off.long()
        cnt = po[1:] - po[:-1]
        owner = torch.repeat_interleave(torch.arange(nb, device="cuda"), cnt)
        dist = tick[owner] - tick[dp.preds[: int(po[-1])].long()]
        mind = torch.full((nb,), 1 << 40, dtype=torch.long, device="cuda").scatter_reduce(0, owner, dist, "amin")
        has = cnt > 0
        d = mind[has].float()
        qs = torch.quantile(d[: 2**24], torch.tensor([0.001, 0.01, 0.05, 0.5], device="cuda")).tolist()
        print(f"lag {lag}: blocks {nb} with preds {int(has.sum())}; nearest-pred ticket distance "
              f"q0.1%={qs[0]:.0f} q1%={qs[1]:.0f} q5%={qs[2]:.0f} median={qs[3]:.0f} min={int(d.min())}; "
              f"<1000: {int((d < 1000).sum())} <2000: {int((d < 2000).sum())}")


if __name__ == "__main__":
    main()

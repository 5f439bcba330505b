"""Paired forward-simulation probe: one C2-shaped graph, one removal set, `--runs` paired runs
through the C-ABI; prints per-stage device time. Used under ncu for the simulate kernels:
  ncu --set full --import-source on --clock-control none -k regex:'realize|hop_kernel|count_kernel|seed_kernel' \
      -o gpurun_out/sim python tools/simulate_probe.py --no-warmup
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1702_05854_b200 import capi, hostapi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--edge-factor", type=float, default=16.0)
    ap.add_argument("--runs", type=int, default=31)
    ap.add_argument("--removed", type=int, default=1000)
    ap.add_argument("--kind", type=int, default=0)
    ap.add_argument("--no-warmup", action="store_true")
    args = ap.parse_args()
    g = hostapi.Graph.rmat(args.scale, args.edge_factor, seed=1)
    p_of = g.random_suspects(g.n // 100, seed=2)
    off, src, cum, _, _ = g.arrays()
    rng = np.random.Generator(np.random.PCG64(1))
    limit = g.m if args.kind == 0 else g.n
    ids = np.unique(rng.integers(0, limit, size=args.removed)).astype(np.uint32)
    with capi.Context(0) as ctx:
        ctx.upload_graph(g.n, g.m, off, src, cum, p_of)
        if not args.no_warmup:
            ctx.paired_runs(args.kind, ids, 7, min(args.runs, 8))
        ctx.stage_times(reset=True)
        l0 = ctx.launches
        t0 = time.perf_counter()
        full, res, _ = ctx.paired_runs(args.kind, ids, 7, args.runs)
        wall = time.perf_counter() - t0
        ms, regions = ctx.stage_times(reset=True)["simulate"]
        draws = args.runs * (g.n + int(np.count_nonzero(p_of)))
        print(json.dumps({"n": g.n, "m": g.m, "runs": args.runs, "wall_s": wall,
                          "layout": os.environ.get("HSAW_LAYOUT", "default"),
                          "device_ms": ms, "batches": regions, "launches": ctx.launches - l0,
                          "draws": draws, "gdraws_per_s_device": draws / ms / 1e6,
                          "mean_full": float(full.mean()), "mean_residual": float(res.mean())}))


if __name__ == "__main__":
    main()

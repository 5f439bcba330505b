import os, sys, time, traceback
sys.path.insert(0, os.getcwd())
import torch
from paper_1702_05854_b200 import capi, hostapi
from paper_1702_05854_b200.sharded import Comm, GpuEngine, ShardedSolver
g = hostapi.Graph.rmat(20, 16.0, seed=1)
p_of = g.random_suspects(g.n // 100, seed=2)
off, src, cum, _, _ = g.arrays()
with capi.Context(0) as ctx:
    ctx.upload_graph(g.n, g.m, off, src, cum, p_of)
    for it in range(2):
        eng = GpuEngine(ctx, seed=42, cfg=capi.SamplerCfg(max_attempts=10**15))
        try:
            t0 = time.perf_counter()
            res = ShardedSolver(eng, Comm()).interdict(g.n, 0, 100, 0.1, 1.0 / g.n)
            print(time.perf_counter() - t0, res["iterations"], res["samples_used"], res["coverage"], res["solution"][:5])
        except Exception:
            traceback.print_exc()
        finally:
            eng.close()

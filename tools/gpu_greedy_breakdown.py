"""Dev script: per-kernel time of one greedy call at a given scale (uses ncu-free CUDA events by
running each phase through the public API and reading stage timers)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_05854_b200 import capi, hostapi
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 23
walks = int(sys.argv[2]) if len(sys.argv) > 2 else 8_000_000
g = hostapi.Graph.rmat(scale, 16, seed=1)
p_of = g.random_suspects(max(1, g.n // 100), seed=2)
dg = hostapi.DeviceGraph(g, p_of)
ctx = capi.Context.borrow(dg.ctx_handle(), g.n, g.m)
with ctx.stream(seed=42, cfg=capi.SamplerCfg(max_attempts=10**15)) as st:
    st.ensure(walks)
    for kind in (0, 1):
        for rep in range(2):
            ctx.stage_times(reset=True)
            t = time.time()
            sol, cov = ctx.greedy(100, stream=st, kind=kind, off=0, cnt=walks)
            wall = time.time() - t
            stg = ctx.stage_times(reset=True)
            print(json.dumps(dict(kind=kind, rep=rep, walks=walks, wall_ms=round(wall * 1e3, 2), cov=cov,
                                  stages={k: round(v[0], 2) for k, v in stg.items() if v[1]})), flush=True)
dg.close()

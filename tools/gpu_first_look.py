"""Dev script: timing look at the sampler / greedy stages and the eSIA host loop on an R-MAT shape.
Usage: python tools/gpu_first_look.py [scale] [batches] [esia_k]   (env knobs: HSAW_L2_FETCH,
HSAW_K1_BLOCKS_PER_SM)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1702_05854_b200 import capi, hostapi

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
esia_k = int(sys.argv[3]) if len(sys.argv) > 3 else 100
tag = {k: os.environ.get(k) for k in ("HSAW_L2_FETCH", "HSAW_K1_BLOCKS_PER_SM") if os.environ.get(k)}
t = time.time()
g = hostapi.Graph.rmat(scale, 16, seed=1)
p_of = g.random_suspects(max(1, g.n // 100), seed=2)
print(f"graph n={g.n} m={g.m} gen {time.time()-t:.1f}s knobs={tag}", flush=True)
t = time.time()
dg = hostapi.DeviceGraph(g, p_of)
print(f"upload {time.time()-t:.3f}s", flush=True)
ctx = capi.Context.borrow(dg.ctx_handle(), g.n, g.m)
for rep in range(3):
    with ctx.stream(seed=42, cfg=capi.SamplerCfg(max_attempts=10**12)) as st:
        st.collect_stats(os.environ.get("LOOK_STATS", "0") == "1")
        ctx.stage_times(reset=True)
        t = time.time()
        acc = st.sample_range(0, nb)
        wall = time.time() - t
        stg = ctx.stage_times(reset=True)
        stats = st.stats()
        if not stats["steps"]:
            ws = ctx.encode_stats(42, nb)
            stats["steps"], stats["alg_bytes"] = ws["steps"], ws["alg_bytes"]
            ctx.stage_times(reset=True)
        k1 = stg["encode"][0] / 1e3
        if rep:
            print(json.dumps(dict(rep=rep, accepted=acc, wall_ms=round(wall * 1e3, 2),
                                  stages_ms={k: round(v[0], 3) for k, v in stg.items() if v[1]},
                                  k1_Gsteps=round(stats["steps"] / k1 / 1e9, 2),
                                  k1_alg_GBs=round(stats["alg_bytes"] / k1 / 1e9, 1),
                                  
                                  hsaw_per_s_wall=round(acc / wall / 1e6, 2), replayed=stats['spare'],
                                  dropped=stats['dropped'])), flush=True)
for rep in range(3):
    ctx.stage_times(reset=True)
    r = hostapi.interdict(g, p_of, 0, esia_k, 0.1, 1.0 / g.n, seed=42, max_attempts=10**15, dg=dg,
                          want_json=True)
    stg = ctx.stage_times(reset=True)
    print("alloc", capi.alloc_counters())
    print(json.dumps(dict(esia_rep=rep, timing={k: round(v, 4) for k, v in r["timing"].items()},
                          it=r["iterations"], samples=r["samples_used"], cov=r["coverage"],
                          stages_ms={k: round(v[0], 2) for k, v in stg.items() if v[1]})), flush=True)
t = time.time()
with hostapi.DeviceGraph(g, p_of) as dg2:
    t1 = time.time()
    at, ac = dg2.sample(1_500_000, seed=7, max_attempts=10**15)
    t2 = time.time()
print(json.dumps(dict(e2e_upload_s=round(t1 - t, 4), e2e_sample_s=round(t2 - t1, 4),
                      e2e_total_s=round(time.time() - t, 4), accepted=ac)))
dg.close()

"""Dev script: first timing look at the sampler and greedy stages on the C2 R-MAT shape."""
import json
import sys
import time
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1702_05854_b200 import capi, rmat

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
t = time.time()
g = rmat.rmat_graph(scale, 16)
print(f"graph n={g.n} m={g.m} gen {time.time()-t:.1f}s", flush=True)
with capi.Context(0) as ctx:
    t = time.time()
    ctx.upload_graph(g.n, g.m, g.in_offsets, g.in_src, g.in_cum, g.p_of)
    print(f"upload {time.time()-t:.3f}s graph_bytes={ctx.graph_bytes/1e6:.1f} MB", flush=True)
    for rep in range(3):
        with ctx.stream(seed=42, cfg=capi.SamplerCfg(max_attempts=10**12)) as st:
            ctx.stage_times(reset=True)
            t = time.time()
            acc = st.sample_range(0, nb)
            wall = time.time() - t
            stg = ctx.stage_times(reset=True)
            stats = st.stats()
            k1 = stg["encode"][0] / 1e3
            print(json.dumps(dict(rep=rep, batches=nb, accepted=acc, wall_s=round(wall, 4),
                                  stages_ms={k: round(v[0], 3) for k, v in stg.items()},
                                  stats=stats,
                                  k1_steps_per_s=stats["steps"] / k1 if k1 else None,
                                  k1_alg_GBs=stats["alg_bytes"] / k1 / 1e9 if k1 else None,
                                  hsaw_per_s_wall=acc / wall)), flush=True)
            if rep == 2:
                size = acc // 2
                for kind in (0, 1):
                    ctx.stage_times(reset=True)
                    t = time.time()
                    sol, cov = ctx.greedy(100, stream=st, kind=kind, off=0, cnt=size)
                    c2 = ctx.coverage_of(sol, stream=st, kind=kind, off=size, cnt=size)
                    wall = time.time() - t
                    stg = ctx.stage_times(reset=True)
                    print(json.dumps(dict(greedy_kind=kind, walks=size, cov=cov, cov_rp=c2,
                                          wall_s=round(wall, 4), sol_head=sol[:5].tolist(),
                                          stages_ms={k: round(v[0], 3) for k, v in stg.items()})),
                          flush=True)
    print("launches", ctx.launches)

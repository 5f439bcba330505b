"""Where an eSIA solve spends its device time: stage timers of one warm run on a bench workload.
python tools/esia_stages.py [c4|c2|c3] [k]   (also prints how concentrated the edge-record touches of
accepted walks are: the share of all touches that the hottest 60 MB / 600 MB of records receive)"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1702_05854_b200 import capi, hostapi  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
sh = bench.WORKLOADS[name]
k = int(sys.argv[2]) if len(sys.argv) > 2 else sh["k"]
p_of = hostapi.random_suspects_n(sh["n"], max(1, sh["n"] // 100), bench.SUSPECT_SEED)
dg = hostapi.DeviceGraph.from_rmat(sh["n"], sh["raw"], bench.GEN_SEED, p_of)
g = dg.graph
ctx = capi.Context.borrow(dg.ctx_handle(), g.n, g.m)
import os
REPS = int(os.environ.get("REPS", "2"))
for rep in range(REPS):
    ctx.stage_times(reset=True)
    t0 = time.perf_counter()
    r = hostapi.interdict(g, p_of, 0, k, 0.1, 1.0 / g.n, seed=42, max_attempts=10**15, dg=dg,
                          want_json=True)
    wall = time.perf_counter() - t0
    st = ctx.stage_times(reset=True)
    try:
        alloc = capi.alloc_counters()
    except Exception:
        alloc = None
    print(json.dumps({"rep": rep, "wall_s": round(wall, 3), "alloc": alloc, "timing": r["timing"],
                      "iterations": r["iterations"], "samples_used": r["samples_used"],
                      "coverage": r["coverage"],
                      "stage_ms": {n_: round(v[0], 1) for n_, v in st.items() if v[1]},
                      "stage_launches": {n_: v[1] for n_, v in st.items() if v[1]}}), flush=True)

# touch concentration of the 32-byte edge records (one record is read per walk step)
if os.environ.get("NO_TOUCH"):
    dg.close()
    sys.exit(0)
with ctx.stream(seed=42, cfg=capi.SamplerCfg(max_attempts=10**15)) as s:
    s.keep(nodes=False, edges=True)
    s.ensure(1_000_000)
    pool = s.export(0, 1_000_000, nodes=False)
cnt = np.bincount(pool.edges, minlength=g.m)
coc = np.bincount(cnt)                      # records with a given touch count
mass = coc * np.arange(coc.size)            # touches they receive
order = np.arange(coc.size)[::-1]
rec_cum, mass_cum = np.cumsum(coc[order]), np.cumsum(mass[order])
total = int(mass.sum())
out = {"sampled_touches": total, "records": int(g.m), "records_touched": int((cnt > 0).sum())}
for mb in (60, 600, 6000):
    nrec = mb * (1 << 20) // 32
    i = int(np.searchsorted(rec_cum, nrec))
    share = float(mass_cum[min(i, mass_cum.size - 1)]) / total
    out[f"share_of_touches_in_hottest_{mb}MB"] = round(share, 4)
print(json.dumps(out))
dg.close()

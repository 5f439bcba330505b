"""Edge counts after dedupe of the device R-MAT generator for the named shapes (bench.WORKLOADS):
python tools/rmat_calibrate.py c3 c4 [raw_edges]"""
import json
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1702_05854_b200 import capi, hostapi  # noqa: E402

names = [a for a in sys.argv[1:] if a in bench.WORKLOADS]
raws = [int(a) for a in sys.argv[1:] if a.isdigit()]
for name in names:
    sh = bench.WORKLOADS[name]
    raw = raws[0] if raws else sh["raw"]
    t0 = time.perf_counter()
    dg = hostapi.DeviceGraph.from_rmat(sh["n"], raw, bench.GEN_SEED, None)
    dt = time.perf_counter() - t0
    ctx = capi.Context.borrow(dg.ctx_handle(), dg.graph.n, dg.graph.m)
    print(json.dumps({"shape": name, "n": dg.graph.n, "raw": raw, "m": dg.graph.m,
                      "kept": dg.graph.m / raw, "build_s": round(dt, 3), "layout": ctx.graph_layout,
                      "graph_bytes": ctx.graph_bytes, "upload_ms": ctx.stage_times()["upload"]}),
          flush=True)
    dg.close()

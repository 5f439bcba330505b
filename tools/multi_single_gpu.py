"""The C++ multi-device solve (host/multi.cpp) with a repeated device id — the only way to run it on
a one-GPU box: ranks share cuda:0 and exchange in process instead of over NCCL. Times eSIA against
the single-device solve on the same host arrays and checks the results are identical.
python tools/multi_single_gpu.py [c2|c3|c4] [k] [ranks] [multi|single]"""
import json
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1702_05854_b200 import hostapi  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 100
ranks = int(sys.argv[3]) if len(sys.argv) > 3 else 2
sh = bench.WORKLOADS[name]
p_of = hostapi.random_suspects_n(sh["n"], max(1, sh["n"] // 100), bench.SUSPECT_SEED)
dg = hostapi.DeviceGraph.from_rmat(sh["n"], sh["raw"], bench.GEN_SEED, p_of, want_host=True)
g = dg.graph
dg.close()
keys = ("solution", "coverage", "attempts", "samples_used", "iterations", "est_suspension")
out = {"workload": name, "n": g.n, "m": g.m, "k": k, "transport": hostapi.multi_transport([0] * ranks)}
only = sys.argv[4] if len(sys.argv) > 4 else ""  # "multi" / "single": run just that arm (memory)
for label, fn in (
        ("single", lambda: hostapi.interdict(g, p_of, 0, k, 0.1, 1.0 / g.n, seed=42, max_attempts=10**15)),
        (f"multi_{ranks}x_cuda0", lambda: hostapi.interdict_devices(g, p_of, 0, k, 0.1, 1.0 / g.n, [0] * ranks,
                                                                    seed=42, max_attempts=10**15,
                                                                    with_timing=True))):
    if only and not label.startswith(only):
        continue
    runs = []
    for _ in range(2):
        t0 = time.perf_counter()
        r = fn()
        runs.append(time.perf_counter() - t0)
    out[label] = {"seconds_first": round(runs[0], 3), "seconds": round(runs[1], 3),
                  "timing": r.get("timing"),
                  **{k_: r[k_] for k_ in keys if k_ != "solution"}, "solution_head": r["solution"][:5]}
    out.setdefault("_results", []).append({k_: r[k_] for k_ in keys})
out["identical"] = len(out["_results"]) == 2 and out["_results"][0] == out["_results"][1]
del out["_results"]
print(json.dumps(out))

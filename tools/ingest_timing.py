"""Cache ingest timing at C2 shape: host load_cache (+ upload) vs device ingest (the reference's own loader is timed by `bench.py --ingest`, cpu_baseline leg)."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1702_05854_b200 import hostapi  # noqa: E402


def best(fn, reps=3):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        ts.append(time.perf_counter() - t0)
        if hasattr(r, "close"):
            r.close()
        del r
    return min(ts)


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    g = hostapi.Graph.rmat(scale, 16.0, seed=1)
    p_of = g.random_suspects(g.n // 100, seed=2)
    with tempfile.TemporaryDirectory(dir="/dev/shm" if os.path.isdir("/dev/shm") else None) as tmp:
        path = os.path.join(tmp, "g.hsaw1")
        g.save_cache(path)
        size = os.path.getsize(path)
        out = {"n": g.n, "m": g.m, "file_bytes": size}
        out["host_load_cache_s"] = best(lambda: hostapi.Graph.load_cache(path))
        h = hostapi.Graph.load_cache(path)
        out["host_upload_s"] = best(lambda: hostapi.DeviceGraph(h, p_of))
        out["device_load_cache_s"] = best(lambda: hostapi.Graph.load_cache_device(path))
        out["device_from_cache_s"] = best(lambda: hostapi.DeviceGraph.from_cache(path))
    out["file_to_resident_speedup_vs_host_path"] = (
        (out["host_load_cache_s"] + out["host_upload_s"]) / out["device_from_cache_s"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()

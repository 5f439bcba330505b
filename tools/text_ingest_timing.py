"""Edge-list text ingest timing at C2 shape: host load_edge_list vs load_edge_list_device (the reference's own
loader is timed by `bench.py --ingest`, cpu_baseline leg).
The file is what save_edge_list writes ("u v %.17g"), read back in 1/in-degree mode."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1702_05854_b200 import hostapi  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    kind = sys.argv[2] if len(sys.argv) > 2 else "synth"
    # validate() rejects R-MAT hub rows in 1/d mode, so the timed file is a uniform
    # graph of the same node / edge count unless "rmat" is asked for
    g = (hostapi.Graph.rmat(scale, 16.0, seed=1) if kind == "rmat"
         else hostapi.Graph.synth(1 << scale, 16, 3))
    with tempfile.TemporaryDirectory(dir="/dev/shm" if os.path.isdir("/dev/shm") else None) as tmp:
        path = os.path.join(tmp, "g.edges")
        g.save_edge_list(path)
        out = {"n": g.n, "m": g.m, "file_bytes": os.path.getsize(path), "graph": kind}
        t0 = time.perf_counter()
        for _ in range(2):
            t0 = time.perf_counter()
            dg = hostapi.DeviceGraph.from_edge_list(path, mode=1)
            out["device_text_to_resident_graph_s"] = time.perf_counter() - t0
            if dg is not None:
                dg.close()
        for name, fn in (("device_load_edge_list_s", hostapi.Graph.load_edge_list_device),
                         ("device_load_edge_list_2nd_s", hostapi.Graph.load_edge_list_device),
                         ("host_load_edge_list_s", hostapi.Graph.load_edge_list)):
            t0 = time.perf_counter()
            try:
                fn(path, mode=1)
                out[name] = time.perf_counter() - t0
            except hostapi.HsawError as e:
                out[name] = time.perf_counter() - t0
                out[name.replace("_s", "_error")] = str(e)[:120]
    print(json.dumps(out))


if __name__ == "__main__":
    main()

"""build_graph: host C++ (the reference's algorithm, hsaw::build_graph) vs the device builder
(hsaw::build_graph_device / hsaw_gpu_graph_build_upload) on the edge list of the bench graph.
Run on the GPU box: python tools/build_timing.py [scale]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1702_05854_b200 import capi, hostapi  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = hostapi.Graph.rmat(scale, 16.0, seed=1)
off, src, cum, _, dst = g.arrays()
perm = np.random.default_rng(1).permutation(g.m)
u, v = np.ascontiguousarray(src[perm]), np.ascontiguousarray(dst[perm])
p_of = g.random_suspects(max(1, g.n // 100), seed=2)
print(f"n={g.n} m={g.m}")
try:
    t0 = time.perf_counter()
    gh = hostapi.Graph.build(g.n, u, v, None, 1)
    print(f"host build_graph (C++, 1 thread): {time.perf_counter() - t0:.3f} s")
except Exception as e:  # hub rows: validate() rejects d >= 36217
    print(f"host build_graph: {time.perf_counter() - t0:.3f} s until it threw: {str(e)[:80]}")
for it in range(3):
    t0 = time.perf_counter()
    try:
        gd = hostapi.Graph.build_device(g.n, u, v, None, 1)
        o2, s2, c2, _, _ = gd.arrays()
        same = np.array_equal(o2, off) and np.array_equal(s2, src) and c2.tobytes() == cum.tobytes()
        print(f"device build_graph_device (ProbGraph back on the host): {time.perf_counter() - t0:.3f} s, identical={same}")
    except Exception as e:
        print(f"device build_graph_device: {time.perf_counter() - t0:.3f} s until it threw: {str(e)[:80]}")
with capi.Context(0) as ctx:
    for it in range(3):
        t0 = time.perf_counter()
        try:
            ctx.build_upload_graph(g.n, u, v, p_of, None, 1)
            print(f"device build + install (no host CSR): {1e3 * (time.perf_counter() - t0):.2f} ms")
        except Exception as e:
            print(f"device build + install: {1e3 * (time.perf_counter() - t0):.2f} ms until it threw: {str(e)[:80]}")
    t0 = time.perf_counter()
    ctx.upload_graph(g.n, g.m, off, src, cum, p_of)
    print(f"upload of the ready CSR: {1e3 * (time.perf_counter() - t0):.2f} ms")

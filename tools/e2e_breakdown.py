"""Where the host-buffer (e2e) call spends its time: context creation, graph upload, sampling.
Run on the GPU box: python tools/e2e_breakdown.py [scale]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1702_05854_b200 import capi, hostapi  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = hostapi.Graph.rmat(scale, 16.0, seed=1)
p_of = g.random_suspects(max(1, g.n // 100), seed=2)
off, src, cum, _, _ = g.arrays()
print(f"n={g.n} m={g.m} bytes={(off.nbytes + src.nbytes + cum.nbytes + p_of.nbytes) / 1e6:.1f} MB")
for it in range(4):
    t0 = time.perf_counter()
    ctx = capi.Context(0)
    t1 = time.perf_counter()
    ctx.upload_graph(g.n, g.m, off, src, cum, p_of)
    t2 = time.perf_counter()
    with ctx.stream(seed=42 + it, cfg=capi.SamplerCfg(max_attempts=10**15)) as st:
        st.ensure(1_567_000)
        t3 = time.perf_counter()
        at, ac = st.counters_for(1_567_000)
    t4 = time.perf_counter()
    ctx.close()
    t5 = time.perf_counter()
    print(f"iter {it}: ctx_create {1e3*(t1-t0):.2f} ms, upload {1e3*(t2-t1):.2f} ms, ensure "
          f"{1e3*(t3-t2):.2f} ms, counters {1e3*(t4-t3):.2f} ms, close {1e3*(t5-t4):.2f} ms, "
          f"total {1e3*(t5-t0):.2f} ms")
for it in range(3):
    t0 = time.perf_counter()
    with hostapi.DeviceGraph(g, p_of, device=0) as dg:
        t1 = time.perf_counter()
        _, acc = dg.sample(1_567_000, seed=100 + it, max_attempts=10**15)
        t2 = time.perf_counter()
    t3 = time.perf_counter()
    print(f"hostapi iter {it}: DeviceGraph {1e3*(t1-t0):.2f} ms, sample {1e3*(t2-t1):.2f} ms, "
          f"close {1e3*(t3-t2):.2f} ms")

"""Where does the L2 flush cost go? Events around the flush and around the sampling step."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1702_05854_b200 import capi, hostapi

g = hostapi.Graph.rmat(20, 16.0, seed=1)
p_of = g.random_suspects(g.n // 100, seed=2)
ts = torch.cuda.Stream()
dg = hostapi.DeviceGraph(g, p_of, device=0, cuda_stream=ts.cuda_stream)
ctx = capi.Context.borrow(dg.ctx_handle(), g.n, g.m)
cfg = capi.SamplerCfg(max_attempts=10**15)
B = 1 << 20
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def step(i):
    with ctx.stream(seed=42, cfg=cfg) as st:
        return st.sample_range(i * B, B)
for mode in ("none", "zero", "read"):
    for i in range(3): step(i)
    torch.cuda.synchronize()
    ctx.stage_times(reset=True)
    tf = tsamp = 0.0
    with torch.cuda.stream(ts):
        for i in range(3, 11):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(ts)
            if mode == "zero": flush.zero_()
            if mode == "read": flush.view(torch.int32).sum()
            e[1].record(ts)
            step(i)
            e[2].record(ts)
            torch.cuda.synchronize()
            tf += e[0].elapsed_time(e[1]); tsamp += e[1].elapsed_time(e[2])
    st = ctx.stage_times(reset=True)
    print(mode, "flush ms", tf / 8, "step ms", tsamp / 8, {k: round(v[0] / 8, 3) for k, v in st.items() if v[1]})

import torch
x = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for name, fn in (("zero_", lambda: x.zero_()), ("sum", lambda: x.view(torch.int32).sum())):
        for _ in range(3): fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(10): fn()
        b.record(s); torch.cuda.synchronize()
        print(name, a.elapsed_time(b) / 10, "ms")

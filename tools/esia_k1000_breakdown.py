import sys, time, json
sys.path.insert(0, '/root/repo')
from paper_1702_05854_b200 import hostapi
g = hostapi.Graph.rmat(20, 16.0, seed=1)
p_of = g.random_suspects(g.n // 100, seed=2)
with hostapi.DeviceGraph(g, p_of) as dg:
    for rep in range(3):
        dg.stage_times(reset=True)
        l0 = dg.launches()
        r = hostapi.interdict(g, p_of, 0, 1000, 0.1, 1.0 / g.n, seed=42, max_attempts=10**15, dg=dg, want_json=True)
        st = dg.stage_times(reset=True)
        print(json.dumps({"timing": r["timing"], "iters": r["iterations"], "launches": dg.launches() - l0,
                          "stages": {k: (round(v[0], 2), v[1]) for k, v in st.items() if v[1]}}))

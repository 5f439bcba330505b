#!/usr/bin/env python
"""Full-size parity fixture (BASELINE.json configs[1], "C2"): the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference/proj/src by oracle/Makefile) solves eSIA k=100, nSIA k=100 and eSIA
k=1000 on the bench's own C2 arrays (R-MAT scale 20, edge factor 16, generator seed 1, 1/in-degree
weights, n/100 random suspects seed 2, stream seed 42, eps 0.1, delta 1/n).

Written to tests/golden/c2_reference.json: InterdictionResult fields + the reference's wall time
and the host cores used (the CPU seconds-to-solution the bench line quotes beside the GPU's),
plus a digest of R_t u R'_t of the last eSIA iteration (the fixed walk set the final greedy ran
on), so that tests can check the device pool is that walk set before comparing greedy outputs.

Takes minutes of CPU (the reference builds a vector<vector> CoverageIndex of m entries per
iteration). Run here (no GPU needed):  python tests/golden/make_c2_golden.py
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from oracle.oracle import Csr  # noqa: E402
from paper_1702_05854_b200 import hostapi  # noqa: E402


def pool_digest(pool, count):
    """sha256 over the first `count` walks of a pool: lengths, nodes, edge ids."""
    eo = pool.edge_off.astype(np.uint64)[: count + 1]
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(eo).tobytes())
    h.update(np.ascontiguousarray(pool.nodes[: int(eo[-1]) + count]).tobytes())
    h.update(np.ascontiguousarray(pool.edges[: int(eo[-1])]).tobytes())
    return h.hexdigest()


def main():
    assert oracle.have_ref(), "oracle/_ref missing: run oracle.build() where /root/reference exists"
    R = oracle.Ref()
    g = hostapi.Graph.rmat(20, 16.0, seed=1)
    p_of = g.random_suspects(g.n // 100, seed=2)
    off, src, cum, _, _ = g.arrays()
    csr = Csr(g.n, g.m, off, src, cum, p_of)
    workers = os.cpu_count() or 1
    out = {"graph": {"rmat_scale": 20, "edge_factor": 16.0, "gen_seed": 1, "n": g.n, "m": g.m,
                     "suspects": g.n // 100, "suspect_seed": 2},
           "stream_seed": 42, "epsilon": 0.1, "delta": 1.0 / g.n, "workers": workers,
           "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": \t")}
    with R.handles(csr) as hd:
        for name, kind, k in (("esia_k100", 0, 100), ("nsia_k100", 1, 100), ("esia_k1000", 0, 1000)):
            t0 = time.perf_counter()
            r = R.interdict(csr, kind, k, 0.1, 1.0 / g.n, seed=42, workers=workers,
                            max_attempts=10**15, hd=hd, want_json=True)
            r["reference_wall_time_s"] = r.pop("wall_time_s")
            r.pop("json")
            r["call_s"] = time.perf_counter() - t0
            out[name] = r
            print(name, {k_: v for k_, v in r.items() if k_ != "solution"}, flush=True)
        # the walk set of the final eSIA k=100 iteration: the stream's first samples_used walks
        su = out["esia_k100"]["samples_used"]
        pool = R.stream_samples(csr, su, seed=42, workers=workers, max_attempts=10**15, hd=hd)
        assert pool.nsamples >= su
        out["esia_k100"]["walkset_sha256"] = pool_digest(pool, su)
        eo = pool.edge_off.astype(np.int64)
        out["esia_k100"]["walkset_items"] = int(eo[su])
        # north_star mode 1 at real size: the reference's greedy on R_t (first half), fixed walk set
        half = su // 2
        t0 = time.perf_counter()
        sol, cov = R.greedy(g.m, eo[: half + 1], pool.edges[: eo[half]], 100, kind=0)
        out["esia_k100"]["greedy_on_rt"] = {"solution": [int(x) for x in sol], "coverage": int(cov),
                                            "seconds": time.perf_counter() - t0}
        assert out["esia_k100"]["greedy_on_rt"]["solution"] == out["esia_k100"]["solution"]
    with open(os.path.join(ROOT, "tests", "golden", "c2_reference.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("written")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Golden vectors for the ranking baselines, produced by the UNMODIFIED
reference's baseline() (proj/src/evaluation.cpp:330-395 through oracle/ref_shim.cpp) on the graph of
tests/golden/partition_vectors.npz: every kind x mode x k, with the PrgState after the call (which
pins the number of draws rr_node_sets consumed). -> tests/golden/baseline_vectors.json"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from oracle.oracle import Csr, OracleError  # noqa: E402


def main():
    R = oracle.Ref()
    pv = np.load(os.path.join(ROOT, "tests", "golden", "partition_vectors.npz"))
    n = pv["in_offsets"].size - 1
    csr = Csr(n, pv["in_src"].size, pv["in_offsets"], pv["in_src"], pv["in_cum"], pv["p_of"])
    s0 = R.seed_from_worker(9)
    out = {"state0": s0, "infmax_samples": 3000, "cases": []}
    with R.handles(csr) as hd:
        for kind in ("randomized", "maxdegree", "pagerank", "infmax-v", "infmax-vi"):
            for mode in (1, 0):
                for k in (1, 7, 70):
                    try:
                        ids, s = R.baseline(csr, kind, mode, k, s0, 3000, hd=hd)
                        out["cases"].append(dict(kind=kind, mode=mode, k=k, ids=ids, state=s))
                    except OracleError as e:
                        out["cases"].append(dict(kind=kind, mode=mode, k=k, error=str(e)))
    with open(os.path.join(ROOT, "tests", "golden", "baseline_vectors.json"), "w") as f:
        json.dump(out, f)
    print(len(out["cases"]), "cases")


if __name__ == "__main__":
    main()

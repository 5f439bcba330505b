"""Generates tests/golden/evaluation_vectors.json by running the UNMODIFIED reference
(oracle/_ref: lt_forward_simulate / estimate_suspension of proj/src/evaluation.cpp, reached through
oracle/ref_shim.cpp) in the build container. Usage:  python tests/golden/make_eval_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Csr, Ref  # noqa: E402
from paper_1702_05854_b200 import rmat  # noqa: E402


def _hexlist(xs):
    return np.array([float.fromhex(x) for x in xs], dtype=np.float64)


def graphs():
    g = json.load(open(os.path.join(HERE, "reference_vectors.json")))
    fx = g["fixture12_given"]
    f12 = Csr(fx["n"], fx["m"], np.array(fx["in_offsets"], dtype=np.uint64),
              np.array(fx["in_src"], dtype=np.uint32), _hexlist(fx["in_cum"]), _hexlist(fx["p_of"]))
    c1 = g["config1_indegree"]["seed42"]
    f12i = Csr(f12.n, f12.m, f12.in_offsets, f12.in_src, _hexlist(c1["in_cum"]), _hexlist(c1["p_of"]))
    z = np.load(os.path.join(HERE, "synth3000.npz"))
    s3 = Csr(z["in_offsets"].size - 1, z["in_src"].size, z["in_offsets"], z["in_src"], z["in_cum"],
             z["p_of"])
    r = rmat.rmat_graph(13, 12.0, seed=5, suspect_frac=0.02, suspect_seed=6)
    r13 = Csr(r.n, r.m, r.in_offsets, r.in_src, r.in_cum, r.p_of)
    return {"fixture12_given": f12, "config1_indegree": f12i, "synth3000": s3,
            "rmat13 (rmat_graph(13, 12.0, seed=5, suspect_frac=0.02, suspect_seed=6))": r13}


def removal_sets(csr):
    rng = np.random.Generator(np.random.PCG64(99))
    edge = sorted(set(int(x) for x in rng.integers(0, csr.m, size=min(40, max(3, csr.m // 6)))))
    node = sorted(set(int(x) for x in rng.integers(0, csr.n, size=min(25, max(2, csr.n // 5)))))
    return [(0, edge), (1, node), (0, edge[:1]), (1, node[:1]), (0, [])]


def main():
    R = Ref()
    out = {}
    for name, csr in graphs().items():
        rec = {"n": csr.n, "m": csr.m}
        with R.handles(csr) as hd:
            st = R.seed_from_worker(7)
            seq = []
            s = st
            for _ in range(6):  # chained calls on one PrgState (evaluation.hpp:25-26)
                cnt, s = R.lt_forward_simulate(csr, s, hd=hd)
                seq.append(cnt)
            rec["lt_forward_simulate"] = dict(state0=st, infected=seq, state_after=s)
            ests = []
            for kind, ids in removal_sets(csr):
                for eps, delta in ((0.3, 0.2), (0.15, 0.05)):
                    if csr.n > 5000 and eps < 0.2:
                        continue
                    e = R.estimate_suspension(csr, kind, ids, eps, delta, st, hd=hd)
                    ests.append(dict(kind=kind, ids=ids, epsilon=eps, delta=delta, state0=st,
                                     value=float.hex(e["value"]), capped=e["capped"],
                                     runs=e["runs"], state_after=e["state"]))
            rec["estimate_suspension"] = ests
        out[name] = rec

    # draw cap (evaluation.cpp:17,229): a removal that never changes the outcome — an edge into a
    # node... any edge whose source is unreachable from every suspect — leaves the sum at 0 until
    # max_runs = 10^9 / (|V_I| + n) runs are spent.
    name = "synth3000"
    csr = graphs()[name]
    deg_in = np.diff(csr.in_offsets.astype(np.int64))
    # an edge out of a node with no in-edges that is not a suspect can never carry infection
    dead_src = np.flatnonzero((deg_in == 0) & (csr.p_of == 0))
    ids = [int(e) for e in np.flatnonzero(np.isin(csr.in_src, dead_src))[:3]]
    if ids:
        st = R.seed_from_worker(11)
        e = R.estimate_suspension(csr, 0, ids, 0.3, 0.2, st)
        out[name]["capped_case"] = dict(kind=0, ids=ids, epsilon=0.3, delta=0.2, state0=st,
                                        value=float.hex(e["value"]), capped=e["capped"],
                                        runs=e["runs"], state_after=e["state"])
    with open(os.path.join(HERE, "evaluation_vectors.json"), "w") as f:
        json.dump(out, f, indent=1)
    print({k: (len(v["estimate_suspension"]), v.get("capped_case", {}).get("runs")) for k, v in out.items()})


if __name__ == "__main__":
    main()

"""Golden vectors for the device CSR builder, generated with the compiled reference (oracle/_ref)
in the build container: build_graph (proj/src/graph.cpp:112-199) on seeded random edge lists.
Writes tests/golden/build_graph.npz. Run: python tests/golden/make_build_golden.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle  # noqa: E402


def edge_list(n, ne, seed, hub=None):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, size=ne, dtype=np.int64)
    v = rng.integers(0, n, size=ne, dtype=np.int64)
    if hub is not None:  # a high in-degree row: long sequential cumulative sum
        extra = np.arange(1, hub + 1, dtype=np.int64) % n
        u = np.concatenate([u, extra])
        v = np.concatenate([v, np.zeros(hub, dtype=np.int64)])
    keep = u != v
    u, v = u[keep], v[keep]
    key = np.unique(v * n + u, return_index=True)[1]
    key.sort()
    u, v = u[key], v[key]
    perm = rng.permutation(u.size)  # input order is arbitrary
    return u[perm].astype(np.uint32), v[perm].astype(np.uint32)


def main():
    oracle.build()
    R = oracle.Ref()
    out = {}
    cases = {"indeg_small": (300, 2500, 11, None, 1), "indeg_hub": (5000, 20000, 12, 4000, 1),
             "given": (400, 3000, 13, None, 0)}
    for name, (n, ne, seed, hub, mode) in cases.items():
        u, v = edge_list(n, ne, seed, hub)
        w = None
        if mode == 0:
            rng = np.random.default_rng(seed + 100)
            indeg = np.bincount(v, minlength=n).astype(np.float64)
            w = rng.uniform(0.05, 1.0, size=u.size) / indeg[v]  # row sums <= 1
        gh = R.build_graph(n, u, v, w, mode=mode)
        csr = R._to_csr(gh)
        wt, dst = R.graph_extra(gh)
        R.graph_free(gh)
        out[f"{name}_n"] = np.array([n], dtype=np.uint32)
        out[f"{name}_mode"] = np.array([mode], dtype=np.int32)
        out[f"{name}_u"], out[f"{name}_v"] = u, v
        if w is not None:
            out[f"{name}_w"] = w
        out[f"{name}_off"], out[f"{name}_src"] = csr.in_offsets, csr.in_src
        out[f"{name}_cum"], out[f"{name}_weight"], out[f"{name}_dst"] = csr.in_cum, wt, dst
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "build_graph.npz"), **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()

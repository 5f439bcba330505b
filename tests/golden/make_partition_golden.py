#!/usr/bin/env python
"""Golden vectors for partitioned sampling, produced by the UNMODIFIED
reference (oracle/_ref: proj/src/partition.cpp + sampler.cpp:510-539 through oracle/ref_shim.cpp):
partition_graph (Hash / LabelProp) + extend_partition(h) and distributed_sample on an R-MAT graph
of 3000 nodes with 60 suspects. -> tests/golden/partition_vectors.npz
Run here (reference tree present):  python tests/golden/make_partition_golden.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from oracle.oracle import Csr  # noqa: E402
from paper_1702_05854_b200 import hostapi  # noqa: E402

N, RAW, GEN_SEED, NSUS, P, TARGET, SEED = 3000, 40000, 3, 60, 4, 700, 7


def main():
    assert oracle.have_ref()
    R = oracle.Ref()
    g = hostapi.Graph.rmat_n(N, RAW, seed=GEN_SEED)
    off, src, cum, _, _ = g.arrays()
    p_of = g.random_suspects(NSUS, 2)
    csr = Csr(g.n, g.m, off, src, cum, p_of)
    out = {"in_offsets": off, "in_src": src, "in_cum": cum, "p_of": p_of,
           "params": np.array([N, RAW, GEN_SEED, NSUS, P, TARGET, SEED], dtype=np.int64)}
    with R.handles(csr) as hd:
        for method in ("hash", "labelprop"):
            for hops in (0, 1, 2):
                part = R.partition(csr, P, method, seed=5, hops=hops, hd=hd)
                key = f"{method}_h{hops}"
                out[f"{key}_assign"] = part.assign
                out[f"{key}_extended"] = np.packbits(np.stack(part.extended), axis=1)
                for workers in (1, 3):
                    r = R.distributed_sample(csr, part, TARGET, seed=SEED, workers=workers, hd=hd)
                    if workers == 1:
                        first = r
                    else:  # the reference's own worker-count independence
                        assert (r.crossings, r.attempts, r.targets) == (first.crossings, first.attempts, first.targets)
                        assert np.array_equal(r.pool.nodes, first.pool.nodes)
                r = first
                out[f"{key}_scalars"] = np.array([r.crossings, r.attempts], dtype=np.uint64)
                out[f"{key}_fraction"] = np.array([r.crossing_fraction])
                out[f"{key}_targets"] = np.array(r.targets, dtype=np.uint64)
                for f in ("edge_off", "nodes", "edges", "tag_worker", "tag_seq"):
                    out[f"{key}_pool_{f}"] = getattr(r.pool, f)
                print(key, r.pool.nsamples, r.crossings, r.attempts, r.targets)
        # uneven parts (external assignment): quotas by largest remainder, a zero-quota part
        assign = np.zeros(N, dtype=np.uint32)
        assign[N // 2:] = 1
        assign[-3:] = 2
        assign[-1] = 3
        part = R.partition(csr, 4, "external", assign=assign, hops=1, hd=hd)
        r = R.distributed_sample(csr, part, 101, seed=11, hd=hd)
        out["ext_assign"] = assign
        out["ext_scalars"] = np.array([r.crossings, r.attempts], dtype=np.uint64)
        out["ext_targets"] = np.array(r.targets, dtype=np.uint64)
        for f in ("edge_off", "nodes", "edges", "tag_worker", "tag_seq"):
            out[f"ext_pool_{f}"] = getattr(r.pool, f)
        print("ext", r.pool.nsamples, r.crossings, r.attempts, r.targets)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "partition_vectors.npz"), **out)


if __name__ == "__main__":
    main()

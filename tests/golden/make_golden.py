"""Generates tests/golden/*.json|npz by running the UNMODIFIED reference (oracle/_ref, built from
/root/reference/proj/src by oracle/Makefile) in the build container. The reference cannot travel
to the GPU box, so its outputs are committed here as small fixtures; this script is the record of
how they were made. Usage:  python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Ref  # noqa: E402

REFDATA = "/root/reference/proj/data"


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def pool_record(pool, full: bool):
    rec = dict(nsamples=pool.nsamples, attempts=int(pool.attempts),
               total_edges=int(pool.edge_off[-1]),
               sha256=digest(pool.edge_off, pool.nodes, pool.edges, pool.tag_worker, pool.tag_seq))
    if full:
        rec.update(edge_off=pool.edge_off.tolist(), nodes=pool.nodes.tolist(),
                   edges=pool.edges.tolist(), tag_worker=pool.tag_worker.tolist(),
                   tag_seq=pool.tag_seq.tolist())
    return rec


def main():
    R = Ref()
    out = {}

    # ---- fixture12 (proj/data/fixture12.{edges,suspects}), given weights and suspects file
    gh = R.load_edge_list(f"{REFDATA}/fixture12.edges", mode=0)
    p = R.load_suspects(f"{REFDATA}/fixture12.suspects", gh)
    csr = R._to_csr(gh, p)
    weight, edge_dst = R.graph_extra(gh)
    fx = dict(n=csr.n, m=csr.m, in_offsets=csr.in_offsets.tolist(), in_src=csr.in_src.tolist(),
              in_cum=[float.hex(float(x)) for x in csr.in_cum],
              p_of=[float.hex(float(x)) for x in csr.p_of],
              weight=[float.hex(float(x)) for x in weight], edge_dst=edge_dst.tolist())
    # the reference test-suite's own byte-stable CLI golden (proj/tests/test_cli.cpp:242-251)
    fx["interdict12_json_text"] = open("/root/reference/proj/tests/golden/interdict12.json").read()
    with R.handles(csr) as hd:
        kats = []
        for w in list(range(40, 60)) + [0, 1, 2**63, 2**64 - 1]:
            seeds, lens = R.thread_sample(csr, w, 10, hd=hd)
            walks = []
            for s_, l_ in zip(seeds, lens):
                dec = R.decode(csr, int(s_), int(l_), hd=hd)
                walks.append(dict(seed=int(s_), len=int(l_),
                                  nodes=None if dec is None else dec[0].tolist(),
                                  edges=None if dec is None else dec[1].tolist()))
            kats.append(dict(worker_id=w, seed_state=R.seed_from_worker(w), walks=walks))
        fx["thread_sample"] = kats
        fx["window_variants"] = []
        for heur, win in [(0, 0), (0, 1), (0, 3), (0, 8), (2, 0), (2, 2), (1, 2)]:
            seeds, lens = R.thread_sample(csr, 42, 50, heuristic=heur, window=win, hd=hd)
            fx["window_variants"].append(dict(heuristic=heur, window=win, seeds=seeds.tolist(),
                                              lens=lens.tolist()))
        fx["pool_seed42_target200"] = pool_record(
            R.stream_samples(csr, 200, seed=42, workers=3, hd=hd), full=True)
        # end-to-end golden of the reference's own test-suite (tests/golden/interdict12.json)
        fx["interdict_edge_k3"] = R.interdict(csr, 0, 3, 0.3, 0.2, seed=42, hd=hd)
        fx["interdict_node_k2"] = R.interdict(csr, 1, 2, 0.3, 0.2, seed=42, hd=hd)
        fx["interdict_edge_k3_cand"] = dict(
            cand=[1, 3, 6, 11, 17, 19],
            result=R.interdict(csr, 0, 3, 0.3, 0.2, seed=7, cand=[1, 3, 6, 11, 17, 19], hd=hd))
    out["fixture12_given"] = fx

    # ---- BASELINE config 1: fixture12, 1/in-degree weights, 10 random suspects
    gh = R.load_edge_list(f"{REFDATA}/fixture12.edges", mode=1)
    c1 = {}
    for seed in (42, 0):
        p = R.random_suspects(gh, 10, seed)
        csr = R._to_csr(gh, p)
        c1[f"seed{seed}"] = dict(
            in_cum=[float.hex(float(x)) for x in csr.in_cum],
            p_of=[float.hex(float(x)) for x in csr.p_of],
            esia_k10=R.interdict(csr, 0, 10, 0.1, 0.1, seed=seed),
            nsia_k5=R.interdict(csr, 1, 5, 0.1, 0.1, seed=seed))
    out["config1_indegree"] = c1

    # ---- prng known answers (beyond proj/tests/test_prng.cpp)
    prng = dict(splitmix=[], xorshift=[], seed_from_worker=[], pick=[])
    st = 0
    for _ in range(5):
        st, o = R.splitmix_next(st)
        prng["splitmix"].append([st, o])
    s = 1
    for _ in range(5):
        s, o = R.prg_next(s)
        prng["xorshift"].append([s, o])
    for w in (0, 1, 42, 43, 2**32, 2**64 - 1):
        prng["seed_from_worker"].append([w, R.seed_from_worker(w)])
    for n in (1, 2, 12, 1000, 2**20, 41_700_000, 2**32 - 1):
        s = 0x9E3779B97F4A7C15
        row = []
        for _ in range(8):
            s, v = R.pick_uniform_node(s, n)
            row.append(v)
        prng["pick"].append([n, row])
    out["prng"] = prng

    # ---- schedule / check values (proj/tests/test_coverage.cpp:162-175,213-242 + extra tuples)
    sched = []
    for (M, k, e, d) in [(10, 1, .5, .5), (100, 2, .1, .1), (16085580, 100, .1, 1 / 1048576),
                         (20, 3, .3, .2), (12, 5, .1, .1), (1470000000, 1000, .1, 1 / 41.7e6)]:
        sched.append(dict(M=M, k=k, eps=e, delta=d, **R.schedule(M, k, e, d)))
    out["schedule"] = sched

    # ---- medium synthetic graph: pool + interdiction digests (arrays in the .npz)
    gh = R.synth_graph(3000, 6, 11)
    p = R.random_suspects(gh, 60, 12)
    csr = R._to_csr(gh, p)
    np.savez_compressed(os.path.join(HERE, "synth3000.npz"), in_offsets=csr.in_offsets,
                        in_src=csr.in_src, in_cum=csr.in_cum, p_of=csr.p_of)
    with R.handles(csr) as hd:
        med = dict(n=csr.n, m=csr.m)
        med["pool_seed5_target4000"] = pool_record(
            R.stream_samples(csr, 4000, seed=5, workers=4, hd=hd), full=False)
        batches = []
        for w in range(100, 164):
            seeds, lens = R.thread_sample(csr, w, 10, hd=hd)
            batches.append(dict(worker_id=w, seeds=seeds.tolist(), lens=lens.tolist()))
        med["thread_sample"] = batches
        med["esia_k5"] = R.interdict(csr, 0, 5, 0.2, 0.1, seed=3, workers=4, hd=hd)
        med["nsia_k5"] = R.interdict(csr, 1, 5, 0.2, 0.1, seed=3, workers=4, hd=hd)
    out["synth3000"] = med

    # ---- greedy on raw item sets (the worked micro-instance + random instances with duplicates)
    rng = np.random.Generator(np.random.PCG64(7))
    greedy = []
    for inst in range(12):
        limit = int(rng.integers(8, 60))
        nsets = int(rng.integers(5, 80))
        sizes = rng.integers(0, 7, size=nsets)
        items = rng.integers(0, limit, size=int(sizes.sum())).astype(np.uint32)
        off = np.zeros(nsets + 1, dtype=np.uint64)
        np.cumsum(sizes, out=off[1:])
        cand = None
        if inst % 3 == 1:
            cand = sorted(set(rng.integers(0, limit, size=max(3, limit // 2)).tolist()))
        k = int(min(1 + inst % 8, limit if cand is None else len(cand)))
        sol, cov = R.greedy(limit, off, items, k, cand=cand)
        sol2, cov2 = R.greedy(limit, off, items, k, cand=cand, lazy=False)
        assert sol.tolist() == sol2.tolist() and cov == cov2
        greedy.append(dict(limit=limit, set_off=off.tolist(), items=items.tolist(), cand=cand, k=k,
                           solution=sol.tolist(), coverage=int(cov),
                           coverage_of=int(R.coverage_of(limit, off, items, sol, cand=cand))))
    out["greedy"] = greedy

    with open(os.path.join(HERE, "reference_vectors.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", os.path.join(HERE, "reference_vectors.json"))


if __name__ == "__main__":
    main()

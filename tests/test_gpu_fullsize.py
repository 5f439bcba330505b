"""Parity at BASELINE.json's full size (configs[1], C2: R-MAT scale 20, 16.1 M edges, 1/in-degree
weights, 1 % suspects) through properties that do not need the oracle to replay millions of walks:
layout / chunking independence of the stream (proj/tests/test_sampler.cpp:241-263), the HSAW
invariants of every pooled walk (:230-239), spot checks of random batches against the oracle
(thread_sample + decode, :93-116), and solver results that do not depend on the device layout."""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

B = 1 << 17  # batches per full-size stream (1.3 M attempts, ~200 k walks)


@pytest.fixture(scope="module")
def c2():
    from oracle.oracle import Csr
    from paper_1702_05854_b200 import hostapi
    g = hostapi.Graph.rmat(20, 16.0, seed=1)
    p_of = g.random_suspects(g.n // 100, seed=2)
    off, src, cum, _, dst = g.arrays()
    return g, Csr(g.n, g.m, off, src, cum, p_of), dst


def _digest(pool):
    h = hashlib.sha256()
    for a in (pool.edge_off, pool.nodes, pool.edges, pool.tag_worker, pool.tag_seq):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _sample(gpu_lib, monkeypatch, csr, env, ranges):
    for k in ("HSAW_LAYOUT", "HSAW_FORCE_EXACT", "HSAW_K1_GENERIC", "HSAW_FUSED", "HSAW_PACK"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    with gpu_lib.Context(0) as ctx:
        ctx.upload_graph(csr.n, csr.m, csr.in_offsets, csr.in_src, csr.in_cum, csr.p_of)
        with ctx.stream(seed=42, cfg=gpu_lib.SamplerCfg(max_attempts=10**15)) as st:
            for first, nb in ranges:
                st.sample_range(first, nb)
            return st.export()


def test_stream_is_independent_of_layout_kernel_and_chunking(gpu_lib, monkeypatch, c2):
    _, csr, _ = c2
    whole = [(0, B)]
    ref = _digest(_sample(gpu_lib, monkeypatch, csr, {"HSAW_LAYOUT": "compact"}, whole))
    variants = {
        "fat layout": ({"HSAW_LAYOUT": "fat"}, whole),
        "plain 32-bit sources": ({"HSAW_LAYOUT": "compact", "HSAW_PACK": "0"}, whole),
        "generic K1 on the compact layout": ({"HSAW_LAYOUT": "compact", "HSAW_K1_GENERIC": "1"}, whole),
        "encode + replay instead of recording": ({"HSAW_LAYOUT": "compact", "HSAW_FUSED": "0"}, whole),
        "three uneven ranges": ({"HSAW_LAYOUT": "compact"},
                                [(0, 1000), (1000, B // 3), (1000 + B // 3, B - 1000 - B // 3)]),
    }
    for name, (env, ranges) in variants.items():
        assert _digest(_sample(gpu_lib, monkeypatch, csr, env, ranges)) == ref, name


def test_pooled_walks_are_hsaws_and_match_the_oracle(gpu_lib, monkeypatch, port, c2):
    _, csr, dst = c2
    pool = _sample(gpu_lib, monkeypatch, csr, {}, [(0, B)])
    n_w = pool.nsamples
    assert n_w > 150_000
    eo = pool.edge_off.astype(np.int64)
    lens = np.diff(eo)
    # every edge (id = CSR slot) joins consecutive nodes: in_src[e] is the next node, e lies in the
    # row of the previous one
    walk_of_edge = np.repeat(np.arange(n_w), lens)
    pos = np.arange(eo[-1]) - eo[walk_of_edge]
    prev = pool.nodes[eo[walk_of_edge] + walk_of_edge + pos]
    nxt = pool.nodes[eo[walk_of_edge] + walk_of_edge + pos + 1]
    e = pool.edges[: eo[-1]]
    assert np.array_equal(csr.in_src[e], nxt)
    assert np.array_equal(dst[e], prev)
    # the hit node is a suspect, no earlier node repeats (self-avoidance, checked per walk by sort)
    last = pool.nodes[eo[1:] + np.arange(n_w)]
    assert np.all(csr.p_of[last] > 0)
    key = walk_of_node = np.repeat(np.arange(n_w), lens + 1)
    order = np.lexsort((pool.nodes[: eo[-1] + n_w], key))
    sn, sk = pool.nodes[: eo[-1] + n_w][order], walk_of_node[order]
    assert not np.any((sn[1:] == sn[:-1]) & (sk[1:] == sk[:-1]))
    # (batch, seq) order, and 300 random batches replayed by the oracle
    tags = pool.tag_worker.astype(np.int64) * 16 + pool.tag_seq
    assert np.all(np.diff(tags) > 0)
    rng = np.random.default_rng(7)
    for b in rng.choice(B, size=300, replace=False):
        seeds, ls = port.thread_sample(csr, 42 + int(b), 10)
        mine = np.nonzero(pool.tag_worker == 42 + int(b))[0]
        kept = []
        for s, ln in zip(seeds, ls):
            d = port.decode(csr, int(s), int(ln))
            if d is not None:
                kept.append(d)
        assert len(kept) == len(mine)
        for w, (nodes, edges) in zip(mine, kept):
            assert np.array_equal(pool.walk_nodes(w), nodes)
            assert np.array_equal(pool.walk_edges(w), edges)


@pytest.mark.parametrize("kind,k", [(0, 100), (1, 100)])
def test_solver_result_is_layout_independent(monkeypatch, c2, kind, k):
    from paper_1702_05854_b200 import hostapi
    g, csr, _ = c2
    out = {}
    for layout in ("compact", "fat"):
        monkeypatch.setenv("HSAW_LAYOUT", layout)
        r = hostapi.interdict(g, csr.p_of, kind, k, 0.1, 1.0 / g.n, seed=42, max_attempts=10**15)
        assert r["passed_check"] and len(set(r["solution"])) == k
        assert r["samples_used"] == 2 * (r["samples_used"] // 2)
        out[layout] = r
    assert out["compact"] == out["fat"]


# ---- the reference's own full-size results (tests/golden/make_c2_golden.py: the unmodified
# reference compiled into oracle/_ref solved these on the same C2 arrays, 11 + 5 minutes of CPU)
@pytest.fixture(scope="module")
def c2_golden():
    import json
    import os

    from conftest import GOLDEN_DIR
    with open(os.path.join(GOLDEN_DIR, "c2_reference.json")) as f:
        return json.load(f)


RESULT_KEYS = ("solution", "coverage", "attempts", "samples_used", "iterations", "est_suspension",
               "passed_check")


@pytest.mark.parametrize("layout", ["compact", "fat"])
@pytest.mark.parametrize("name,kind,k", [("esia_k100", 0, 100), ("nsia_k100", 1, 100),
                                         ("esia_k1000", 0, 1000)])
def test_solver_equals_the_reference_at_full_size(monkeypatch, c2, c2_golden, layout, name, kind, k):
    """interdiction.cpp:12-67 end to end at BASELINE configs[1]: every InterdictionResult field the
    reference produced, bit for bit (est_suspension included: same FP64 expression on the host)."""
    from paper_1702_05854_b200 import hostapi
    g, csr, _ = c2
    gold = c2_golden[name]
    assert (c2_golden["graph"]["n"], c2_golden["graph"]["m"]) == (g.n, g.m)
    monkeypatch.setenv("HSAW_LAYOUT", layout)
    r = hostapi.interdict(g, csr.p_of, kind, k, 0.1, 1.0 / g.n, seed=42, max_attempts=10**15)
    for key in RESULT_KEYS:
        assert r[key] == gold[key], key


@pytest.mark.parametrize("name,kind,k", [("esia_k100", 0, 100), ("nsia_k100", 1, 100),
                                         ("esia_k1000", 0, 1000)])
def test_solver_on_dense_instances_equals_the_reference(monkeypatch, c2, c2_golden, name, kind, k):
    """The same full-size goldens with every greedy run forced onto the dense reduced instance
    (greedy.cu build_dense; production switches to it from 256 MB of counters, i.e. above C2):
    thresholded index, renamed items, (start, length) walks, rank -> id mapping of the solution."""
    from paper_1702_05854_b200 import hostapi
    g, csr, _ = c2
    gold = c2_golden[name]
    monkeypatch.setenv("HSAW_DENSE_MIN_BYTES", "0")
    r = hostapi.interdict(g, csr.p_of, kind, k, 0.1, 1.0 / g.n, seed=42, max_attempts=10**15)
    for key in RESULT_KEYS:
        assert r[key] == gold[key], key


def test_fixed_walk_set_greedy_at_full_size(gpu_lib, monkeypatch, c2, c2_golden):
    """north_star's mode 1 at real size: the device pool IS the reference's walk set of the last
    eSIA iteration (sha256 over lengths, nodes and edge ids of 7.7 M walks / 360 M items), and the
    device greedy on R_t (its first half) selects the reference's k edges with the same coverage."""
    import hashlib
    g, csr, _ = c2
    gold = c2_golden["esia_k100"]
    su = gold["samples_used"]
    for k_ in ("HSAW_LAYOUT", "HSAW_FORCE_EXACT", "HSAW_PACK"):
        monkeypatch.delenv(k_, raising=False)
    with gpu_lib.Context(0) as ctx:
        ctx.upload_graph(csr.n, csr.m, csr.in_offsets, csr.in_src, csr.in_cum, csr.p_of)
        with ctx.stream(seed=42, cfg=gpu_lib.SamplerCfg(max_attempts=10**15)) as st:
            st.ensure(su)
            pool = st.export(0, su)
            h = hashlib.sha256()
            h.update(np.ascontiguousarray(pool.edge_off.astype(np.uint64)).tobytes())
            h.update(np.ascontiguousarray(pool.nodes).tobytes())
            h.update(np.ascontiguousarray(pool.edges).tobytes())
            assert int(pool.edge_off[-1]) == gold["walkset_items"]
            assert h.hexdigest() == gold["walkset_sha256"]
            sol, cov = ctx.greedy(100, stream=st, kind=0, off=0, cnt=su // 2)
            assert sol.tolist() == gold["greedy_on_rt"]["solution"] == gold["solution"]
            assert cov == gold["greedy_on_rt"]["coverage"] == gold["coverage"]

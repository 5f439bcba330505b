"""GPU parity tests for the sampler (kernels K1, K2, K2b and the stream), through the C-ABI.
Bar: bit-exact with the oracle — same (seed, len) per batch, same decoded nodes/edges, same pool
order, tags, attempts. Mirrors proj/tests/test_sampler.cpp."""
import hashlib

import os

import numpy as np
import pytest

from conftest import make_csr, upload

pytestmark = pytest.mark.gpu


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def oracle_batches(port, csr, first, nb, l=10, heuristic=0, window=2):
    out = []
    tot = np.zeros(4, dtype=np.uint64)
    for b in range(nb):
        s, ln, st = port.thread_sample(csr, (first + b) % 2**64, l, heuristic=heuristic,
                                       window=window, want_stats=True)
        out.append((s, ln))
        tot += st
    return out, tot


def check_encode(ctx, gpu_lib, port, csr, first, nb, l=10, heuristic=0, window=2):
    cfg = gpu_lib.SamplerCfg(heuristic=heuristic, window=window, batch_size=l)
    seeds, lens, counts, stats = ctx.encode_batches(first, nb, cfg)
    exp, tot = oracle_batches(port, csr, first, nb, l, heuristic, window)
    for b in range(nb):
        c = int(counts[b])
        assert c == len(exp[b][0]), f"batch {b}: count {c} != {len(exp[b][0])}"
        assert seeds[b, :c].tolist() == exp[b][0].tolist(), f"batch {b} seeds"
        assert lens[b, :c].tolist() == exp[b][1].tolist(), f"batch {b} lens"
    assert stats["attempts"] == int(tot[0])
    assert stats["draws"] == int(tot[1])
    assert stats["steps"] == int(tot[2])
    assert stats["alg_bytes"] == int(tot[3])
    assert stats["accepted"] == int(counts.sum())


def small_graphs():
    from paper_1702_05854_b200 import rmat
    return {
        "uniform2000": rmat.uniform_graph(2000, 5, seed=3, suspect_count=40, suspect_seed=4),
        "rmat12": rmat.rmat_graph(12, 8, seed=3, suspect_frac=0.02),
        "rmat14_dense": rmat.rmat_graph(14, 24, seed=5, suspect_frac=0.01),
    }


def test_encode_golden_kats(ctx, gpu_lib, golden, fixture12):
    """Device K1 against the reference's own outputs (fixtures), no oracle in the loop."""
    upload(ctx, fixture12)
    for kat in golden["fixture12_given"]["thread_sample"]:
        seeds, lens, counts, _ = ctx.encode_batches(kat["worker_id"], 1)
        c = int(counts[0])
        assert seeds[0, :c].tolist() == [w["seed"] for w in kat["walks"]]
        assert lens[0, :c].tolist() == [w["len"] for w in kat["walks"]]
    for v in golden["fixture12_given"]["window_variants"]:
        cfg = gpu_lib.SamplerCfg(heuristic=v["heuristic"], window=v["window"], batch_size=50)
        seeds, lens, counts, _ = ctx.encode_batches(42, 1, cfg)
        c = int(counts[0])
        assert seeds[0, :c].tolist() == v["seeds"] and lens[0, :c].tolist() == v["lens"]


def test_unknown_heuristic_is_rejected(ctx, gpu_lib, fixture12):
    upload(ctx, fixture12)
    with pytest.raises(gpu_lib.HsawError) as e:
        ctx.encode_batches(0, 1, gpu_lib.SamplerCfg(heuristic=3))
    assert e.value.status == gpu_lib.HSAW_EINVAL


@pytest.mark.parametrize("name,window", [("uniform2000", 2), ("uniform2000", 0), ("rmat12", 2),
                                         ("rmat14_dense", 3), ("ring", 0)])
def test_encode_floyd_matches_oracle(ctx, gpu_lib, port, name, window):
    """CycleHeuristic::Floyd (proj/src/sampler.cpp:113-138): the tortoise cursor replays the
    attempt's draw stream on the device; batches equal the oracle's, work counters included (the
    tortoise's draws are not the attempt's: sampler.cpp:128-133 uses the second cursor's state)."""
    if name == "ring":  # cycles only: every walk that misses the single suspect is flagged
        from oracle.oracle import Csr
        n = 64
        p = np.zeros(n)
        p[0] = 0.02
        csr = Csr(n, n, np.arange(n + 1, dtype=np.uint64),
                  ((np.arange(n) + 1) % n).astype(np.uint32), np.ones(n), p)
    else:
        csr = make_csr(small_graphs()[name])
    upload(ctx, csr)
    check_encode(ctx, gpu_lib, port, csr, 77, 600, l=10, heuristic=1, window=window)


def test_encode_matches_oracle_fixture12(ctx, gpu_lib, port, fixture12, fixture12_indegree):
    upload(ctx, fixture12)
    check_encode(ctx, gpu_lib, port, fixture12, 0, 300)
    check_encode(ctx, gpu_lib, port, fixture12, 2**64 - 100, 200)  # worker id wraps (u64)
    upload(ctx, fixture12_indegree)
    check_encode(ctx, gpu_lib, port, fixture12_indegree, 42, 300)


@pytest.mark.parametrize("name", ["uniform2000", "rmat12", "rmat14_dense"])
def test_encode_matches_oracle(ctx, gpu_lib, port, name):
    g = small_graphs()[name]
    csr = make_csr(g)
    upload(ctx, csr)
    check_encode(ctx, gpu_lib, port, csr, 1000, 1500)


def test_encode_synth3000_golden(ctx, golden, synth3000):
    upload(ctx, synth3000)
    b0 = golden["synth3000"]["thread_sample"]
    seeds, lens, counts, _ = ctx.encode_batches(b0[0]["worker_id"], len(b0))
    for i, b in enumerate(b0):
        c = int(counts[i])
        assert seeds[i, :c].tolist() == b["seeds"] and lens[i, :c].tolist() == b["lens"]


@pytest.mark.parametrize("heuristic,window,l", [(0, 0, 10), (0, 1, 7), (0, 3, 10), (0, 8, 10),
                                                (2, 0, 10), (2, 2, 25), (0, 2, 1), (0, 2, 100)])
def test_encode_config_variants(ctx, gpu_lib, port, heuristic, window, l):
    g = small_graphs()["uniform2000"]
    csr = make_csr(g)
    upload(ctx, csr)
    check_encode(ctx, gpu_lib, port, csr, 5, 400, l=l, heuristic=heuristic, window=window)


def test_encode_given_weights_total_below_one(ctx, gpu_lib, port):
    """Rows whose weights are non-uniform and sum to < 1: the 'no live edge' branch and the
    binary-search fallback of the pick (interpolation guess misses) both run."""
    rng = np.random.Generator(np.random.PCG64(11))
    n, d = 600, 40
    off = np.arange(0, n * d + 1, d, dtype=np.uint64)
    src = np.empty(n * d, dtype=np.uint32)
    cum = np.empty(n * d, dtype=np.float64)
    for v in range(n):
        cand = np.setdiff1d(rng.choice(n, size=d + 1, replace=False), [v])[:d]
        src[v * d:(v + 1) * d] = np.sort(cand)
        w = rng.random(d) ** 4 + 1e-9
        w = w / w.sum() * rng.uniform(0.3, 0.95)
        c = 0.0
        for j in range(d):
            c += float(w[j])
            cum[v * d + j] = c
    p = np.zeros(n)
    p[rng.choice(n, size=30, replace=False)] = rng.uniform(0.15, 1.0, size=30)
    from oracle.oracle import Csr
    csr = Csr(n, n * d, off, src, cum, p)
    upload(ctx, csr)
    check_encode(ctx, gpu_lib, port, csr, 0, 800)


def test_encode_high_degree_hub(ctx, gpu_lib, port):
    """A 1/d star with d = 50000 (> 36217: total weight drifts above 1) plus a feeder ring:
    interpolation guess on a huge row, total > 1, empty rows."""
    from paper_1702_05854_b200 import rmat
    d = 50000
    n = d + 1
    u = np.concatenate([np.arange(1, n, dtype=np.uint64), np.zeros(200, dtype=np.uint64)])
    v = np.concatenate([np.zeros(d, dtype=np.uint64), np.arange(1, 201, dtype=np.uint64)])
    off, src = rmat.csr_from_edges(n, u, v)
    cum = rmat.indegree_cum(off)
    assert cum[d - 1] > 1.0
    p = np.zeros(n)
    p[np.arange(300, n, 997)] = 0.5
    from oracle.oracle import Csr
    csr = Csr(n, int(off[-1]), off, src, cum, p)
    upload(ctx, csr)
    check_encode(ctx, gpu_lib, port, csr, 0, 600)


# ---- decode -------------------------------------------------------------------------------------
def test_decode_matches_oracle(ctx, gpu_lib, port):
    g = small_graphs()["uniform2000"]
    csr = make_csr(g)
    upload(ctx, csr)
    seeds, lens, counts, _ = ctx.encode_batches(0, 600)
    enc = [(int(seeds[b, j]), int(lens[b, j])) for b in range(600) for j in range(int(counts[b]))]
    eo, nodes, edges, status = ctx.decode_walks([e[0] for e in enc], [e[1] for e in enc])
    dropped = 0
    for w, (s, ln) in enumerate(enc):
        exp = port.decode(csr, s, ln)
        if exp is None:
            assert status[w] == 0
            dropped += 1
            continue
        assert status[w] == 1
        a, b = int(eo[w]), int(eo[w + 1])
        assert nodes[a + w:b + w + 1].tolist() == exp[0].tolist()
        assert edges[a:b].tolist() == exp[1].tolist()
    assert dropped > 0  # the exact recheck must have something to do on this graph


def test_decode_golden_fixture12(ctx, golden, fixture12):
    upload(ctx, fixture12)
    walks = [w for kat in golden["fixture12_given"]["thread_sample"] for w in kat["walks"]]
    eo, nodes, edges, status = ctx.decode_walks([w["seed"] for w in walks],
                                                [w["len"] for w in walks])
    for i, w in enumerate(walks):
        if w["nodes"] is None:
            assert status[i] == 0
        else:
            a, b = int(eo[i]), int(eo[i + 1])
            assert status[i] == 1
            assert nodes[a + i:b + i + 1].tolist() == w["nodes"]
            assert edges[a:b].tolist() == w["edges"]


def test_decode_foreign_encodings(ctx, port, fixture12):
    """proj/tests/test_sampler.cpp:118-124: a (seed, len) that no walk has is a replay mismatch;
    the oracle's verdict (DataError vs dropped) must be reproduced per walk."""
    from oracle.oracle import OracleError
    upload(ctx, fixture12)
    seeds = [0xABCDEF, 0, 12345, 99, 7, 0xDEADBEEF, 424242, 31337] * 8
    lens = [7, 3, 0, 1, 2, 11, 5, 4] * 8
    seeds = [s + i for i, s in enumerate(seeds)]
    seeds[1] = 0
    _, _, _, status = ctx.decode_walks(seeds, lens)
    for i, (s, ln) in enumerate(zip(seeds, lens)):
        try:
            exp = port.decode(fixture12, s, ln)
            want = 0 if exp is None else 1
        except OracleError:
            want = 2
        assert status[i] == want, (i, s, ln)


def test_cyclic_walks_decode_to_nothing(ctx, port):
    """proj/tests/test_sampler.cpp:126-145: 3-cycle at weight 1 + isolated suspect."""
    from oracle.oracle import Csr
    csr = Csr(4, 3, [0, 1, 2, 3, 3], [2, 0, 1], [1.0, 1.0, 1.0], [0, 0, 0, 1.0])
    upload(ctx, csr)
    seeds, tested = [], 0
    for x in range(1, 2000):
        _, start = port.pick_uniform_node(x, 4)
        if start != 3:
            seeds.append(x)
        if len(seeds) == 200:
            break
    _, _, _, status = ctx.decode_walks(seeds, [4] * len(seeds))
    assert (status == 0).all()


def test_long_walk_distinct_check(ctx, port):
    """Walks longer than the shared-memory hash capacity take the global-table path: a directed
    ring of 6000 nodes with one certain suspect gives self-avoiding walks of up to 5999 edges."""
    from oracle.oracle import Csr
    n = 6000
    off = np.arange(n + 1, dtype=np.uint64)
    src = ((np.arange(n) + 1) % n).astype(np.uint32)
    p = np.zeros(n)
    p[0] = 1.0
    csr = Csr(n, n, off, src, np.ones(n), p)
    upload(ctx, csr)
    with ctx.stream(seed=3, cfg=None) as st:
        st.ensure(300)
        got = st.to_pool(300)
    exp = port.stream_samples(csr, 300, seed=3)
    assert got.attempts == exp.attempts and got.nsamples == exp.nsamples
    assert np.array_equal(got.nodes, exp.nodes) and np.array_equal(got.edges, exp.edges)
    assert int(np.diff(exp.edge_off.astype(np.int64)).max()) > 2048


def test_log_growth_opt_in(ctx, port, monkeypatch):
    """HSAW_LOG_GROW=1 (csrc/sampler.cu grow_log, the generic K1 = the fat layout's production
    kernel): walks that outgrow their 4096-pair log chunk move to a larger run of chunks while
    they are recorded - several times on a ring of 20000 nodes - instead of being replayed by K2.
    Same pool as the oracle; on the fat layout nothing is replayed."""
    from oracle.oracle import Csr
    n = 20000
    off = np.arange(n + 1, dtype=np.uint64)
    src = ((np.arange(n) + 1) % n).astype(np.uint32)
    p = np.zeros(n)
    p[0] = 1.0
    csr = Csr(n, n, off, src, np.ones(n), p)
    upload(ctx, csr)
    exp = port.stream_samples(csr, 60, seed=9)
    assert int(np.diff(exp.edge_off.astype(np.int64)).max()) > 16384
    monkeypatch.setenv("HSAW_LOG_GROW", "1")
    monkeypatch.setenv("HSAW_PIPE_BATCHES", "8")  # small calls: the arena does not run out
    with ctx.stream(seed=9, cfg=None) as st:
        for b in range(0, 64, 8):
            st.sample_range(b, 8)
        pools_equal(st.to_pool(60), exp)
        replayed = st.stats()["spare"]
    if os.environ.get("HSAW_LAYOUT") == "fat":
        assert replayed == 0


# ---- stream -------------------------------------------------------------------------------------
def pools_equal(got, exp):
    assert got.nsamples == exp.nsamples
    assert got.attempts == exp.attempts
    assert np.array_equal(got.edge_off, exp.edge_off)
    assert np.array_equal(got.nodes, exp.nodes)
    assert np.array_equal(got.edges, exp.edges)
    assert np.array_equal(got.tag_worker, exp.tag_worker)
    assert np.array_equal(got.tag_seq, exp.tag_seq)


def test_stream_pool_golden(ctx, golden, fixture12, synth3000):
    upload(ctx, fixture12)
    exp = golden["fixture12_given"]["pool_seed42_target200"]
    with ctx.stream(seed=42) as st:
        st.ensure(200)
        got = st.to_pool(200)
    assert got.attempts == exp["attempts"] and got.nsamples == exp["nsamples"]
    assert got.nodes.tolist() == exp["nodes"] and got.edges.tolist() == exp["edges"]
    assert got.tag_worker.tolist() == exp["tag_worker"] and got.tag_seq.tolist() == exp["tag_seq"]
    upload(ctx, synth3000)
    exp = golden["synth3000"]["pool_seed5_target4000"]
    with ctx.stream(seed=5) as st:
        st.ensure(4000)
        got = st.to_pool(4000)
    assert (got.nsamples, got.attempts) == (exp["nsamples"], exp["attempts"])
    assert digest(got.edge_off, got.nodes, got.edges, got.tag_worker, got.tag_seq) == exp["sha256"]


def test_stream_floyd_matches_oracle(ctx, gpu_lib, port):
    """The whole stream under CycleHeuristic::Floyd: pool, tags and attempts equal the oracle's
    (the unfused K1 -> K2 -> K2b path serves every non-default SamplerConfig)."""
    csr = make_csr(small_graphs()["uniform2000"])
    upload(ctx, csr)
    for window in (2, 0):
        with ctx.stream(seed=8, cfg=gpu_lib.SamplerCfg(heuristic=1, window=window)) as st:
            st.ensure(2500)
            pools_equal(st.to_pool(2500),
                        port.stream_samples(csr, 2500, seed=8, heuristic=1, window=window))


@pytest.mark.parametrize("name", ["uniform2000", "rmat12"])
def test_stream_matches_oracle(ctx, port, name):
    csr = make_csr(small_graphs()[name])
    upload(ctx, csr)
    with ctx.stream(seed=5) as st:
        st.ensure(3000)
        pools_equal(st.to_pool(3000), port.stream_samples(csr, 3000, seed=5))
        # over-materialisation and incremental growth do not change any prefix
        # (proj/tests/test_sampler.cpp:241-263, sampler.hpp:128-132)
        st.ensure(9000)
        pools_equal(st.to_pool(3000), port.stream_samples(csr, 3000, seed=5))
        pools_equal(st.to_pool(7777), port.stream_samples(csr, 7777, seed=5))
        assert st.counters_for(0) == (0, 0)
        acc = st.count
        with pytest.raises(Exception) as e:
            st.counters_for(acc + 1)
        assert e.value.status == 4
        with pytest.raises(Exception) as e:
            st.export(acc - 1, 5)
        assert e.value.status == 4


def test_stream_sample_range_concatenates(ctx, port):
    """Sharding building block: issuing the batch ranges in pieces equals one stream."""
    csr = make_csr(small_graphs()["uniform2000"])
    upload(ctx, csr)
    with ctx.stream(seed=9) as st:
        total = 0
        for first, nb in ((0, 100), (100, 1), (101, 999), (1100, 400)):
            total += st.sample_range(first, nb)
        assert total == st.count
        got = st.export(0, total)
        nb_cut, acc = st.local_cut(total)
        assert acc == total and nb_cut <= 1500
    exp = port.stream_samples(csr, total, seed=9)
    assert exp.nsamples == total
    assert np.array_equal(got.nodes, exp.nodes) and np.array_equal(got.tag_seq, exp.tag_seq)
    assert exp.attempts == nb_cut * 10


def test_stream_budget_exhaustion(ctx, gpu_lib, synth3000):
    """proj/tests/test_sampler.cpp:265-271 -> SamplingError (status 3)."""
    from oracle.oracle import Csr
    csr = Csr(synth3000.n, synth3000.m, synth3000.in_offsets, synth3000.in_src, synth3000.in_cum,
              np.zeros(synth3000.n))
    upload(ctx, csr)
    with ctx.stream(seed=0, cfg=gpu_lib.SamplerCfg(max_attempts=5000)) as st:
        with pytest.raises(gpu_lib.HsawError) as e:
            st.ensure(100)
        assert e.value.status == gpu_lib.HSAW_EBUDGET
        assert st.size()[1] == 500  # floor(5000 / 10) batches were tried


def test_stream_self_avoidance_and_hits(ctx, synth3000):
    upload(ctx, synth3000)
    with ctx.stream(seed=1) as st:
        st.ensure(5000)
        pool = st.export()
    for w in range(pool.nsamples):
        nodes = pool.walk_nodes(w)
        assert len(set(nodes.tolist())) == len(nodes)
        assert synth3000.p_of[nodes[-1]] > 0
        e = pool.walk_edges(w)
        for i in range(len(e)):  # edge e[i] goes nodes[i+1] -> nodes[i]
            assert synth3000.in_src[e[i]] == nodes[i + 1]
            assert synth3000.in_offsets[nodes[i]] <= e[i] < synth3000.in_offsets[nodes[i] + 1]


def test_suspects_reupload(ctx, port, synth3000):
    from oracle.oracle import Csr
    upload(ctx, synth3000)
    rng = np.random.Generator(np.random.PCG64(1))
    p2 = np.zeros(synth3000.n)
    p2[rng.choice(synth3000.n, 25, replace=False)] = rng.uniform(0.2, 1.0, 25)
    ctx.upload_suspects(p2)
    csr2 = Csr(synth3000.n, synth3000.m, synth3000.in_offsets, synth3000.in_src, synth3000.in_cum, p2)
    with ctx.stream(seed=2) as st:
        st.ensure(1500)
        pools_equal(st.to_pool(1500), port.stream_samples(csr2, 1500, seed=2))


def test_upload_rejects_bad_graphs(ctx, gpu_lib):
    with pytest.raises(gpu_lib.HsawError) as e:
        ctx.upload_graph(3, 2, [0, 1, 2, 2], [1, 7], [1.0, 1.0], [0, 0, 1.0])
    assert e.value.status == gpu_lib.HSAW_EDATA  # source id out of range
    with pytest.raises(gpu_lib.HsawError) as e:
        ctx.upload_graph(3, 2, [0, 2, 2, 2], [1, 2], [0.6, 0.4], [0, 0, 1.0])
    assert e.value.status == gpu_lib.HSAW_EDATA  # cumulative weights decrease


def test_upload_beside_the_check_rejects_bad_sources(ctx, gpu_lib, monkeypatch):
    """The layout built beside the in_cum check (segments of sources, csrc/graph.cu) reports a bad
    source row like the plain path does, with the reference's wording."""
    from paper_1702_05854_b200 import rmat
    monkeypatch.setenv("HSAW_UPLOAD_REGEN", "3")
    monkeypatch.setenv("HSAW_UPLOAD_CHUNK_EDGES", "512")
    g = rmat.rmat_graph(12, 10, seed=3, suspect_frac=0.02)
    src = g.in_src.copy()
    row = int(np.argmax(np.diff(g.in_offsets.astype(np.int64))))
    src[int(g.in_offsets[row]) + 1] = g.n + 5
    with pytest.raises(gpu_lib.HsawError) as e:
        ctx.upload_graph(g.n, g.m, g.in_offsets, src, g.in_cum, g.p_of)
    assert e.value.status == gpu_lib.HSAW_EDATA
    assert "source id out of range" in str(e.value) and str(row) in str(e.value)
    ctx.upload_graph(g.n, g.m, g.in_offsets, g.in_src, g.in_cum, g.p_of)  # the context is still usable
    with ctx.stream(seed=1) as st:
        st.ensure(100)


# ---- fused recording path (K1 logs walks while generating them) ---------------------------------
def test_fused_overflow_and_arena_exhaustion(ctx, port, monkeypatch):
    """Walks that outgrow their log chunk, and walks generated after the arena ran out, must be
    replayed by K2 and land in the pool exactly like recorded ones."""
    csr = make_csr(small_graphs()["uniform2000"])
    upload(ctx, csr)
    exp = port.stream_samples(csr, 4000, seed=11)
    monkeypatch.setenv("HSAW_ARENA_MAX_PAIRS", "4096")  # four chunks for thousands of lanes
    with ctx.stream(seed=11) as st:
        st.ensure(4000)
        got = st.to_pool(4000)
        assert st.stats()["spare"] > 0  # some walks took the replay path
    pools_equal(got, exp)
    monkeypatch.delenv("HSAW_ARENA_MAX_PAIRS")
    with ctx.stream(seed=11) as st:
        st.ensure(4000)
        pools_equal(st.to_pool(4000), exp)


def test_pipelined_chunks_match(ctx, port, monkeypatch):
    """A call that spans several chunks samples chunk i + 1 on a second stream while chunk i is
    rechecked and compacted (csrc/stream.cu sample_range). The pool and its order must not depend
    on the cut: tiny chunks (HSAW_PIPE_BATCHES), tiny chunks with the arena running out (replays
    beside chunks sampled ahead), and the serial chunks of HSAW_PIPELINE=0 all give the
    reference's pool (sampler.cpp:423-461: pool order = worker id, then sequence)."""
    csr = make_csr(small_graphs()["uniform2000"])
    upload(ctx, csr)
    exp = port.stream_samples(csr, 6000, seed=13)
    for env in ({"HSAW_PIPE_BATCHES": "64"},
                {"HSAW_PIPE_BATCHES": "37", "HSAW_ARENA_MAX_PAIRS": "4096"},
                {"HSAW_PIPE_BATCHES": "64", "HSAW_PIPELINE": "0"},
                {"HSAW_PIPE_BATCHES": "1"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        with ctx.stream(seed=13) as st:
            st.ensure(6000)
            pools_equal(st.to_pool(6000), exp)
        for k in env:
            monkeypatch.delenv(k)
    # explicit ranges: one pipelined call equals the same range issued batch by batch
    monkeypatch.setenv("HSAW_PIPE_BATCHES", "50")
    with ctx.stream(seed=13) as st:
        st.sample_range(0, 700)
        n_piped = st.count
        piped = st.to_pool(n_piped)
    monkeypatch.delenv("HSAW_PIPE_BATCHES")
    with ctx.stream(seed=13) as st:
        for b in range(700):
            st.sample_range(b, 1)
        n_serial = st.count
        serial = st.to_pool(n_serial)
    assert n_piped == n_serial
    pools_equal(piped, serial)


def test_unfused_path_still_matches(gpu_lib, port, monkeypatch):
    """HSAW_FUSED=0 keeps the encode -> replay pipeline selectable (A/B measurements)."""
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import numpy as np\n"
        "from conftest import make_csr\n"
        "from oracle.oracle import Port\n"
        "from paper_1702_05854_b200 import capi, rmat\n"
        "csr = make_csr(rmat.rmat_graph(12, 8, seed=3, suspect_frac=0.02))\n"
        "exp = Port().stream_samples(csr, 3000, seed=5)\n"
        "with capi.Context(0) as ctx:\n"
        "    ctx.upload_graph(csr.n, csr.m, csr.in_offsets, csr.in_src, csr.in_cum, csr.p_of)\n"
        "    with ctx.stream(seed=5) as st:\n"
        "        st.ensure(3000); got = st.to_pool(3000)\n"
        "assert got.attempts == exp.attempts and np.array_equal(got.nodes, exp.nodes)\n"
        "assert np.array_equal(got.edges, exp.edges) and np.array_equal(got.tag_seq, exp.tag_seq)\n"
        "print('ok')\n"
    ) % (__import__("conftest").ROOT, __import__("os").path.join(__import__("conftest").ROOT, "tests"))
    env = dict(__import__("os").environ, HSAW_FUSED="0")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("threads", ["4", "0"])
def test_large_upload_staged_and_plain(ctx, port, monkeypatch, threads):
    """Uploads of >= 16 MB go through the multi-threaded pinned staging ring (graph.cu,
    StagedCopier); HSAW_UPLOAD_THREADS=0 keeps plain pageable copies. Same pool either way, equal
    to the oracle's stream (proj/src/sampler.cpp:388-463)."""
    from paper_1702_05854_b200 import rmat
    monkeypatch.setenv("HSAW_UPLOAD_THREADS", threads)
    g = rmat.rmat_graph(17, 12, seed=9, suspect_frac=0.01)
    csr = make_csr(g)
    assert 8 * (csr.n + 1) + 12 * csr.m + 8 * csr.n >= 16 << 20
    upload(ctx, csr)
    with ctx.stream(seed=5) as st:
        st.ensure(3000)
        got = st.to_pool(3000)
    exp = port.stream_samples(csr, 3000, seed=5)
    assert got.attempts == exp.attempts and got.nsamples == exp.nsamples
    assert np.array_equal(got.nodes, exp.nodes) and np.array_equal(got.edges, exp.edges)


@pytest.mark.parametrize("weights", ["indegree", "one-bit-off", "given"])
def test_upload_regenerates_indegree_sums(ctx, port, monkeypatch, weights):
    """Large uploads do not send in_cum when host threads have verified, bit for bit, that every
    row holds build_graph's sequential 1/in-degree sums (proj/src/graph.cpp:172-178): the device
    regenerates them. Forced here on a small graph: same pool as the oracle either way, and any
    other weights - a single differing bit included - take the plain copy."""
    from oracle.oracle import Csr
    from paper_1702_05854_b200 import rmat
    monkeypatch.setenv("HSAW_UPLOAD_REGEN", "2")
    g = rmat.rmat_graph(13, 10, seed=4, suspect_frac=0.02)
    cum = g.in_cum.copy()
    if weights == "one-bit-off":  # last bit of one interior cumulative weight (still increasing)
        e = int(np.argmax(np.diff(g.in_offsets.astype(np.int64)))) 
        pos = int(g.in_offsets[e]) + 1
        cum[pos] = np.nextafter(cum[pos], 2.0)
    elif weights == "given":
        deg = np.diff(g.in_offsets.astype(np.int64))
        row = np.repeat(np.arange(g.n), deg)
        cum = cum * (0.5 + 0.4 * ((row % 7) / 7.0))  # rows still increasing, totals below one
    csr = Csr(g.n, g.m, g.in_offsets, g.in_src, cum, g.p_of)
    upload(ctx, csr)
    assert ctx.upload_mode == ("regenerated" if weights == "indegree" else "copied")
    full = 8 * (g.n + 1) + 12 * g.m + 8 * g.n
    assert ctx.upload_bytes == (full - 8 * g.m if weights == "indegree" else full)
    with ctx.stream(seed=6) as st:
        st.ensure(2000)
        got = st.to_pool(2000)
    exp = port.stream_samples(csr, 2000, seed=6)
    assert got.attempts == exp.attempts and got.nsamples == exp.nsamples
    assert np.array_equal(got.nodes, exp.nodes) and np.array_equal(got.edges, exp.edges)


@pytest.mark.parametrize("weights", ["indegree", "one-bit-off"])
def test_upload_shares_indegree_sums_between_check_and_wire(ctx, port, monkeypatch, weights):
    """The check and the link work through in_cum from both ends (RowCheck, csrc/hostcheck.cpp): with
    many small chunks and one check thread some chunks are verified and regenerated, the others
    copied, wherever the two meet. Whatever the split, the device holds the host's exact sums -
    same pool as the oracle - and the bytes sent say how much went over the wire; a differing bit
    anywhere sends everything."""
    from oracle.oracle import Csr
    from paper_1702_05854_b200 import rmat
    monkeypatch.setenv("HSAW_UPLOAD_REGEN", "3")
    monkeypatch.setenv("HSAW_UPLOAD_CHUNK_EDGES", "512")
    monkeypatch.setenv("HSAW_UPLOAD_CHECK_THREADS", "1")
    g = rmat.rmat_graph(14, 10, seed=9, suspect_frac=0.02)
    cum = g.in_cum.copy()
    if weights == "one-bit-off":
        pos = int(g.m) - 2  # in the part the link would take
        cum[pos] = np.nextafter(cum[pos], 0.0) if cum[pos] > cum[pos - 1] else cum[pos]
        if cum[pos] == g.in_cum[pos]:
            pos = int(g.in_offsets[int(np.argmax(np.diff(g.in_offsets.astype(np.int64))))]) + 1
            cum[pos] = np.nextafter(cum[pos], 2.0)
    csr = Csr(g.n, g.m, g.in_offsets, g.in_src, cum, g.p_of)
    upload(ctx, csr)
    base = 8 * (g.n + 1) + 4 * g.m + 8 * g.n
    if weights == "indegree":
        assert base <= ctx.upload_bytes <= base + 8 * g.m
        assert (ctx.upload_bytes - base) % 8 == 0
        assert ctx.upload_mode == ("regenerated" if ctx.upload_bytes < base + 8 * g.m else "copied")
    with ctx.stream(seed=6) as st:
        st.ensure(2000)
        got = st.to_pool(2000)
    exp = port.stream_samples(csr, 2000, seed=6)
    assert got.attempts == exp.attempts and got.nsamples == exp.nsamples
    assert np.array_equal(got.nodes, exp.nodes) and np.array_equal(got.edges, exp.edges)


def test_stream_keeping_one_item_array(ctx, gpu_lib, synth3000, port):
    """hsaw_gpu_stream_keep: a pool that keeps only the edge ids (or only the nodes) has the same
    order and counters, serves greedy / coverage of its own kind bit-exactly, and refuses the other."""
    upload(ctx, synth3000)
    with ctx.stream(seed=11) as both, ctx.stream(seed=11) as eo, ctx.stream(seed=11) as no:
        eo.keep(nodes=False, edges=True)
        no.keep(nodes=True, edges=False)
        for st in (both, eo, no):
            st.ensure(3000)
        assert both.size() == eo.size() == no.size()
        assert both.counters_for(3000) == eo.counters_for(3000) == no.counters_for(3000)
        ref_pool = both.export(0, 3000)
        e_pool = eo.export(0, 3000, nodes=False)
        n_pool = no.export(0, 3000, edges=False)
        assert np.array_equal(e_pool.edges, ref_pool.edges) and np.array_equal(n_pool.nodes, ref_pool.nodes)
        assert np.array_equal(e_pool.edge_off, ref_pool.edge_off)
        for kind, st, other in ((0, eo, no), (1, no, eo)):
            a_sol, a_cov = ctx.greedy(7, stream=st, kind=kind, off=0, cnt=1500)
            b_sol, b_cov = ctx.greedy(7, stream=both, kind=kind, off=0, cnt=1500)
            assert a_sol.tolist() == b_sol.tolist() and a_cov == b_cov
            with pytest.raises(gpu_lib.HsawError) as e:
                ctx.greedy(7, stream=other, kind=kind, off=0, cnt=1500)
            assert e.value.status == gpu_lib.HSAW_EINVAL
        with pytest.raises(gpu_lib.HsawError):
            eo.export(0, 10)
        with pytest.raises(gpu_lib.HsawError):
            eo.keep(nodes=True, edges=True)  # too late: sampling has started

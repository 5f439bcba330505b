"""Paired LT forward simulation on the device against the oracle and the
reference-generated goldens: lt_forward_simulate (proj/src/evaluation.cpp:202-207), the paired run
loop and estimate_suspension (:209-242). Bit-exact: infected counts per run, value/capped/runs and
the PrgState the call leaves behind. Runs on every device layout (conftest.LAYOUTS)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, make_csr, upload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eval_golden():
    with open(os.path.join(GOLDEN_DIR, "evaluation_vectors.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def rmat13():
    from paper_1702_05854_b200 import rmat
    return make_csr(rmat.rmat_graph(13, 12.0, seed=5, suspect_frac=0.02, suspect_seed=6))


@pytest.fixture
def graphs(fixture12, fixture12_indegree, synth3000, rmat13):
    return {"fixture12_given": fixture12, "config1_indegree": fixture12_indegree,
            "synth3000": synth3000, "rmat13": rmat13}


def _golden_for(eval_golden, name):
    for k, v in eval_golden.items():
        if k.split(" ")[0] == name:
            return v
    raise KeyError(name)


def test_lt_forward_simulate_matches_reference(ctx, graphs, eval_golden):
    for name, csr in graphs.items():
        g = _golden_for(eval_golden, name)["lt_forward_simulate"]
        upload(ctx, csr)
        s = g["state0"]
        got = []
        for _ in g["infected"]:
            cnt, s = ctx.lt_forward_simulate(s)
            got.append(cnt)
        assert got == g["infected"], name
        assert s == g["state_after"], name
        # the same runs as one batch on one stream
        full, res, after = ctx.paired_runs(-1, None, g["state0"], len(got))
        assert full.tolist() == g["infected"] and res.tolist() == g["infected"]
        assert after == g["state_after"]


def test_estimate_suspension_matches_reference(ctx, graphs, eval_golden):
    for name, csr in graphs.items():
        g = _golden_for(eval_golden, name)
        upload(ctx, csr)
        cases = list(g["estimate_suspension"])
        if "capped_case" in g:
            cases.append(g["capped_case"])
        for c in cases:
            e = ctx.estimate_suspension(c["kind"], c["ids"], c["epsilon"], c["delta"], c["state0"])
            what = (name, c["kind"], c["ids"][:4], c["epsilon"])
            assert e["runs"] == c["runs"], what
            assert e["capped"] == c["capped"], what
            assert e["value"] == float.fromhex(c["value"]), what
            assert e["state"] == c["state_after"], what


def test_paired_runs_match_oracle_per_run(ctx, graphs, port):
    rng = np.random.Generator(np.random.PCG64(3))
    for name, csr in graphs.items():
        upload(ctx, csr)
        nruns = 300 if csr.n < 100 else 40
        for kind in (0, 1):
            limit = csr.m if kind == 0 else csr.n
            ids = np.unique(rng.integers(0, limit, size=max(2, limit // 8))).astype(np.uint32)
            st = port.seed_from_worker(1000 + kind)
            want_full, want_res, want_state = port.paired_runs(csr, kind, ids, st, nruns)
            full, res, state = ctx.paired_runs(kind, ids, st, nruns)
            assert np.array_equal(full, want_full), (name, kind)
            assert np.array_equal(res, want_res), (name, kind)
            assert state == want_state
            assert np.all(res <= full)
            # a run range that does not start at the stream's origin: chain two calls
            f1, r1, mid = ctx.paired_runs(kind, ids, st, 7)
            f2, r2, end = ctx.paired_runs(kind, ids, mid, nruns - 7)
            assert np.array_equal(np.concatenate([f1, f2]), want_full)
            assert np.array_equal(np.concatenate([r1, r2]), want_res)
            assert end == want_state


def test_hub_rows_and_given_weights(ctx, port):
    """Rows far beyond the linear-scan limit (graph.hpp:67) and rows whose weights sum below 1
    (a draw can land on "no live edge")."""
    from oracle.oracle import Csr
    rng = np.random.Generator(np.random.PCG64(17))
    n = 600
    rows = []
    for v in range(n):
        d = 500 if v == 3 else (40 if v % 50 == 0 else int(rng.integers(0, 6)))
        cand = rng.permutation(n)[: d + 1]
        rows.append(np.sort(cand[cand != v][:d]).astype(np.uint32))
    off = np.zeros(n + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(r) for r in rows])
    src = np.concatenate(rows)
    cum = np.zeros(src.size)
    for v in range(n):
        lo, hi = int(off[v]), int(off[v + 1])
        if hi > lo:
            w = rng.random(hi - lo)
            w *= rng.uniform(0.3, 1.0) / w.sum()
            c = 0.0
            for i in range(lo, hi):  # sequential FP64 sums like build_graph (graph.cpp:158-178)
                c += w[i - lo]
                cum[i] = min(c, 1.0)
    p_of = np.zeros(n)
    p_of[rng.choice(n, 30, replace=False)] = rng.uniform(0.05, 1.0, 30)
    csr = Csr(n, src.size, off, src, cum, p_of)
    upload(ctx, csr)
    st = port.seed_from_worker(5)
    for kind, ids in ((0, np.arange(0, src.size, 7, dtype=np.uint32)), (1, np.array([3, 50, 51], dtype=np.uint32))):
        want = port.paired_runs(csr, kind, ids, st, 60)
        got = ctx.paired_runs(kind, ids, st, 60)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
        assert got[2] == want[2]
        assert ctx.estimate_suspension(kind, ids, 0.3, 0.2, st) == \
            port.estimate_suspension(csr, kind, ids, 0.3, 0.2, st)


def test_argument_errors_follow_the_reference(ctx, fixture12, gpu_lib):
    upload(ctx, fixture12)
    st = 12345
    for eps, delta in ((0.0, 0.1), (1.0, 0.1), (float("nan"), 0.1), (0.1, 0.0), (0.1, 1.0)):
        with pytest.raises(gpu_lib.HsawError) as ei:  # std::invalid_argument, evaluation.cpp:214-217
            ctx.estimate_suspension(0, [1], eps, delta, st)
        assert ei.value.status == gpu_lib.HSAW_EINVAL
    with pytest.raises(gpu_lib.HsawError) as ei:  # DataError, evaluation.cpp:195-200
        ctx.estimate_suspension(0, [1, fixture12.m], 0.3, 0.2, st)
    assert ei.value.status == gpu_lib.HSAW_EDATA
    assert "removal id out of range: %d" % fixture12.m in str(ei.value)
    with pytest.raises(gpu_lib.HsawError) as ei:
        ctx.estimate_suspension(1, [fixture12.n], 0.3, 0.2, st)
    assert ei.value.status == gpu_lib.HSAW_EDATA
    # empty removal: paired runs identical, no draw is consumed (evaluation.cpp:218)
    e = ctx.estimate_suspension(0, [], 0.3, 0.2, st)
    assert e == dict(value=0.0, capped=False, runs=0, state=st)


@pytest.mark.parametrize("layout", ["compact", "fat"])
def test_full_size_runs_match_oracle(gpu_lib, port, monkeypatch, layout):
    """C2 shape (R-MAT scale 20, 16 M edges): two paired runs against the oracle on the L2-resident
    compact layout (the default at this size) and on the fat layout the larger shapes use."""
    from oracle.oracle import Csr
    from paper_1702_05854_b200 import hostapi
    for k in ("HSAW_LAYOUT", "HSAW_FORCE_EXACT", "HSAW_PACK"):
        monkeypatch.delenv(k, raising=False)
    monkeypatch.setenv("HSAW_LAYOUT", layout)
    g = hostapi.Graph.rmat(20, 16.0, seed=1)
    p_of = g.random_suspects(g.n // 100, seed=2)
    off, src, cum, _, _ = g.arrays()
    csr = Csr(g.n, g.m, off, src, cum, p_of)
    rng = np.random.Generator(np.random.PCG64(8))
    ids = np.unique(rng.integers(0, csr.m, size=100000)).astype(np.uint32)
    st = port.seed_from_worker(99)
    want = port.paired_runs(csr, 0, ids, st, 2)
    with gpu_lib.Context(0) as ctx:
        upload(ctx, csr)
        got = ctx.paired_runs(0, ids, st, 2)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
        assert got[2] == want[2]
        # many runs in several device batches: invariants + independence of the batch split
        full, res, end = ctx.paired_runs(0, ids, st, 40)
        assert np.array_equal(full[:2], want[0]) and np.all(res <= full)
        f2, r2, e2 = ctx.paired_runs(0, ids, got[2], 38)
        assert np.array_equal(full[2:], f2) and np.array_equal(res[2:], r2) and e2 == end
        same, same_res, _ = ctx.paired_runs(0, np.zeros(0, dtype=np.uint32), st, 3)
        assert np.array_equal(same, full[:3]) and np.array_equal(same_res, same)


def _two_node():  # proj/tests/oracles.hpp:130-137
    from oracle.oracle import Csr
    return Csr(2, 1, np.array([0, 1, 1], dtype=np.uint64), np.array([1], dtype=np.uint32),
               np.array([0.5]), np.array([0.0, 1.0]))


def test_reference_test_cases(ctx, port):  # proj/tests/test_evaluation.cpp:13-66
    from oracle.oracle import Csr
    chain = Csr(3, 2, np.array([0, 0, 1, 2], dtype=np.uint64), np.array([0, 1], dtype=np.uint32),
                np.array([1.0, 1.0]), np.array([1.0, 0.0, 0.0]))
    upload(ctx, chain)
    full, _, _ = ctx.paired_runs(-1, None, 3, 100)
    assert np.all(full == 3)  # "deterministic chain infects everyone"
    from paper_1702_05854_b200 import rmat
    g = rmat.uniform_graph(30, 3, seed=1, suspect_count=1)
    g.p_of[:] = 0.0  # "no suspects, no infection": a run is n draws, no member draws
    upload(ctx, make_csr(g))
    full, _, after = ctx.paired_runs(-1, None, 5, 100)
    assert np.all(full == 0)
    assert after == port.paired_runs(make_csr(g), 0, [], 5, 100)[2]
    two = _two_node()
    upload(ctx, two)
    runs = 1_000_000  # "two-node mean tends to 1.5", all runs in one call
    full, _, after = ctx.paired_runs(-1, None, 11, runs)
    assert abs(full.mean() - 1.5) < 0.0075
    want = port.paired_runs(two, 0, [], 11, runs)
    assert np.array_equal(full, want[0]) and after == want[2]
    for kind, ids, truth in ((0, [0], 0.5), (1, [1], 1.5), (1, [0], 0.5)):
        e = ctx.estimate_suspension(kind, ids, 0.05, 0.05, 21)
        assert abs(e["value"] - truth) / truth < 0.05
        assert e == port.estimate_suspension(two, kind, ids, 0.05, 0.05, 21)


def test_host_layer_signatures(eval_golden, synth3000):
    """hsaw::lt_forward_simulate / estimate_suspension of the C++ host layer, both the reference
    signatures (g, vi, ...) and the DeviceGraph overloads."""
    from paper_1702_05854_b200 import hostapi
    g = hostapi.Graph.from_csr(synth3000.n, synth3000.m, synth3000.in_offsets, synth3000.in_src,
                               synth3000.in_cum)
    gold = eval_golden["synth3000"]
    f = gold["lt_forward_simulate"]
    with hostapi.DeviceGraph(g, synth3000.p_of) as dg:
        s, got = f["state0"], []
        for _ in f["infected"]:
            cnt, s = hostapi.lt_forward_simulate(g, synth3000.p_of, s, dg=dg)
            got.append(cnt)
        assert got == f["infected"] and s == f["state_after"]
        for c in gold["estimate_suspension"][:4]:
            e = hostapi.estimate_suspension(g, synth3000.p_of, c["kind"], c["ids"], c["epsilon"],
                                            c["delta"], c["state0"], dg=dg)
            assert e == dict(value=float.fromhex(c["value"]), capped=c["capped"], runs=c["runs"],
                             state=c["state_after"])
    cnt, s = hostapi.lt_forward_simulate(g, synth3000.p_of, f["state0"])
    assert cnt == f["infected"][0]
    c = gold["estimate_suspension"][2]
    e = hostapi.estimate_suspension(g, synth3000.p_of, c["kind"], c["ids"], c["epsilon"],
                                    c["delta"], c["state0"])
    assert e["runs"] == c["runs"] and e["value"] == float.fromhex(c["value"])
    with pytest.raises(hostapi.HsawError) as ei:
        hostapi.estimate_suspension(g, synth3000.p_of, 0, [synth3000.m], 0.3, 0.2, 1)
    assert ei.value.status == 2


def test_cli_estimate(tmp_path, fixture12, eval_golden, golden):
    """`hsaw estimate` (proj/src/cli.cpp:162-185): same JSON document as the reference prints."""
    from paper_1702_05854_b200 import hostapi
    fx = golden["fixture12_given"]
    edges = tmp_path / "f12.edges"
    with open(edges, "w") as f:
        for e in range(fx["m"]):
            f.write(f"{fx['in_src'][e]} {fx['edge_dst'][e]} {float.fromhex(fx['weight'][e])!r}\n")
    sus = tmp_path / "f12.suspects"
    with open(sus, "w") as f:
        for v, p in enumerate(fixture12.p_of):
            if p:
                f.write(f"{v} {float(p)!r}\n")
    rem = tmp_path / "removal.txt"
    ids = [1, 5, 7]
    rem.write_text("".join(f"{i}\n" for i in ids))
    out = tmp_path / "est.json"
    rc = hostapi.run_cli(["estimate", "--graph", str(edges), "--weights", "given", "--suspects",
                          str(sus), "--mode", "edge", "--removal", str(rem), "--epsilon", "0.3",
                          "--delta", "0.2", "--seed", "7", "--output", str(out)])
    assert rc == 0
    doc = json.loads(out.read_text())
    # oracle: PrgState s = seed_from_worker(seed) (cli.cpp:173)
    from oracle.oracle import Port
    P = Port()
    want = P.estimate_suspension(fixture12, 0, ids, 0.3, 0.2, P.seed_from_worker(7))
    assert doc == dict(kind="edge", removed=3, epsilon=0.3, delta=0.2, suspension=want["value"],
                       capped=want["capped"], runs=want["runs"])
    assert list(doc) == sorted(doc)  # nlohmann object order
    assert hostapi.run_cli(["estimate", "--graph", str(edges), "--weights", "given", "--suspects",
                            str(sus), "--removal", str(rem), "--epsilon", "1.5"]) == 1
    rem.write_text("999\n")
    assert hostapi.run_cli(["estimate", "--graph", str(edges), "--weights", "given", "--suspects",
                            str(sus), "--removal", str(rem)]) == 2


def test_degenerate_graphs(ctx, port):
    """One node, no edges, no suspects, zero runs: the corner cases of the stream arithmetic."""
    from oracle.oracle import Csr
    one = Csr(1, 0, np.zeros(2, dtype=np.uint64), np.zeros(0, dtype=np.uint32), np.zeros(0),
              np.array([0.75]))
    upload(ctx, one)
    st = port.seed_from_worker(2)
    want = port.paired_runs(one, 1, [0], st, 500)
    got = ctx.paired_runs(1, [0], st, 500)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]) and got[2] == want[2]
    assert ctx.estimate_suspension(1, [0], 0.3, 0.2, st) == port.estimate_suspension(one, 1, [0], 0.3, 0.2, st)
    full, res, after = ctx.paired_runs(1, [0], st, 0)
    assert full.size == 0 and after == st
    iso = Csr(5, 0, np.zeros(6, dtype=np.uint64), np.zeros(0, dtype=np.uint32), np.zeros(0),
              np.array([0.0, 1.0, 0.0, 0.5, 0.0]))
    upload(ctx, iso)
    want = port.paired_runs(iso, 1, [1, 1, 3], st, 64)  # duplicate ids in the removal set
    got = ctx.paired_runs(1, [1, 1, 3], st, 64)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]) and got[2] == want[2]
    assert np.all(got[1] == 0) and np.all(got[0] >= 1)

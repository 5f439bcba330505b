"""GPU parity tests for the drop-in entry points of the C++ host layer: esia / nsia /
stream_samples / the CLI, end to end on the device, against the reference's goldens and the oracle.
Mirrors proj/tests/test_interdiction.cpp and test_cli.cpp:242-251."""
import json

import numpy as np
import pytest

from conftest import _hexlist, make_csr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def host():
    from paper_1702_05854_b200 import hostapi
    hostapi.lib()
    return hostapi


def as_graph(host, csr):
    return host.Graph.from_csr(csr.n, csr.m, csr.in_offsets, csr.in_src, csr.in_cum)


def test_interdict12_golden(host, golden, fixture12):
    """proj/tests/golden/interdict12.json: --seed 42 --k 3 --epsilon 0.3 --delta 0.2, edge mode."""
    g = as_graph(host, fixture12)
    fx = golden["fixture12_given"]
    got = host.interdict(g, fixture12.p_of, 0, 3, 0.3, 0.2, seed=42, want_json=True)
    js = got.pop("json")
    got.pop("timing")
    assert got == fx["interdict_edge_k3"]
    assert js + "\n" == fx["interdict12_json_text"] or js == fx["interdict12_json_text"].rstrip("\n")
    assert host.interdict(g, fixture12.p_of, 1, 2, 0.3, 0.2, seed=42) == fx["interdict_node_k2"]
    c = fx["interdict_edge_k3_cand"]
    assert host.interdict(g, fixture12.p_of, 0, 3, 0.3, 0.2, seed=7, cand=c["cand"]) == c["result"]


def test_config1_golden(host, golden, fixture12_indegree):
    """BASELINE.json configs[0]: fixture12, 1/in-degree weights, 10 random suspects, eSIA k=10."""
    g = as_graph(host, fixture12_indegree)
    c1 = golden["config1_indegree"]["seed42"]
    assert host.interdict(g, fixture12_indegree.p_of, 0, 10, 0.1, 0.1, seed=42) == c1["esia_k10"]
    assert host.interdict(g, fixture12_indegree.p_of, 1, 5, 0.1, 0.1, seed=42) == c1["nsia_k5"]


def test_synth3000_golden(host, golden, synth3000):
    g = as_graph(host, synth3000)
    with host.DeviceGraph(g, synth3000.p_of) as dg:  # one upload, both solvers
        assert host.interdict(g, synth3000.p_of, 0, 5, 0.2, 0.1, seed=3, dg=dg) == \
            golden["synth3000"]["esia_k5"]
        assert host.interdict(g, synth3000.p_of, 1, 5, 0.2, 0.1, seed=3, dg=dg) == \
            golden["synth3000"]["nsia_k5"]
        again = host.interdict(g, synth3000.p_of, 0, 5, 0.2, 0.1, seed=3, dg=dg)
        assert again == golden["synth3000"]["esia_k5"]  # deterministic, stream state not shared


@pytest.mark.parametrize("kind,k", [(0, 7), (1, 4), (0, 40)])
def test_rmat_matches_oracle(host, port, kind, k):
    from paper_1702_05854_b200 import rmat
    csr = make_csr(rmat.rmat_graph(12, 8, seed=3, suspect_frac=0.02))
    g = as_graph(host, csr)
    assert host.interdict(g, csr.p_of, kind, k, 0.2, 0.1, seed=5) == \
        port.interdict(csr, kind, k, 0.2, 0.1, seed=5)


def test_two_node_closed_forms(host):
    """proj/tests/test_interdiction.cpp:13-38: single edge b -> a at 0.5, b a certain suspect."""
    g = host.Graph.build(2, [1], [0], [0.5], mode=host.WEIGHT_GIVEN)
    p = np.array([0.0, 1.0])
    r = host.interdict(g, p, 0, 1, 0.1, 0.1, seed=5)
    assert r["solution"] == [0] and abs(r["est_suspension"] - 0.5) < 0.02
    r = host.interdict(g, p, 1, 1, 0.1, 0.1, seed=6)
    assert r["solution"] == [1] and abs(r["est_suspension"] - 1.5) < 0.05


def test_doubling_discipline(host, port, synth3000):  # test_interdiction.cpp:40-64
    g = as_graph(host, synth3000)
    r = host.interdict(g, synth3000.p_of, 0, 3, 0.25, 0.2, seed=42)
    sched = host.schedule(synth3000.m, 3, 0.25, 0.2)
    assert r["iterations"] <= sched["t_max"]
    assert r["samples_used"] == 2 * (sched["lambda_samples"] << (r["iterations"] - 1))
    assert r == port.interdict(synth3000, 0, 3, 0.25, 0.2, seed=42)


def test_zero_gain_candidates_exhaust_guard(host):  # test_interdiction.cpp:66-82
    g = host.Graph.build(3, [1], [0], [0.5], mode=host.WEIGHT_GIVEN)
    p = np.array([0.0, 1.0, 0.0])
    r = host.interdict(g, p, 1, 1, 0.3, 0.3, seed=2, cand=[2])
    assert r["solution"] == [2] and r["coverage"] == 0 and not r["passed_check"]
    assert r["est_suspension"] == 0.0
    sched = host.schedule(3, 1, 0.3, 0.3)
    assert r["iterations"] <= sched["t_max"] and r["samples_used"] >= sched["n_max"]


def test_argument_validation(host):  # test_interdiction.cpp:84-99
    g = host.Graph.build(2, [1], [0], [0.5], mode=host.WEIGHT_GIVEN)
    p = np.array([0.0, 1.0])
    for kind, k, cand in ((0, 2, None), (0, 0, None), (1, 3, None)):
        with pytest.raises(host.HsawError) as e:
            host.interdict(g, p, kind, k, 0.1, 0.1, cand=cand)
        assert e.value.status == 1
    with pytest.raises(host.HsawError) as e:
        host.interdict(g, p, 0, 1, 0.1, 0.1, cand=[0, 0])  # duplicate candidate id
    assert e.value.status == 2
    with pytest.raises(host.HsawError) as e:
        host.interdict(g, p, 0, 1, 0.1, 0.1, cand=[5])     # out of range
    assert e.value.status == 2
    with pytest.raises(host.HsawError) as e:
        host.interdict(g, p, 0, 1, 1.5, 0.1)               # epsilon domain
    assert e.value.status == 1


def test_budget_exhaustion_is_sampling_error(host, synth3000):
    g = as_graph(host, synth3000)
    with pytest.raises(host.HsawError) as e:
        host.interdict(g, np.zeros(synth3000.n), 0, 2, 0.2, 0.1, max_attempts=5000)
    assert e.value.status == 3


def test_stream_samples_drop_in(host, port, synth3000):
    """Reference-signature stream_samples(g, vi, workers, target, seed): same pool as the oracle."""
    g = as_graph(host, synth3000)
    got = host.stream_samples(g, synth3000.p_of, 2500, seed=9)
    exp = port.stream_samples(synth3000, 2500, seed=9)
    assert got.attempts == exp.attempts and got.nsamples == exp.nsamples
    assert np.array_equal(got.nodes, exp.nodes) and np.array_equal(got.edges, exp.edges)
    assert np.array_equal(got.tag_worker, exp.tag_worker) and np.array_equal(got.tag_seq, exp.tag_seq)
    with host.DeviceGraph(g, synth3000.p_of) as dg:
        assert dg.sample(2500, seed=9) == (exp.attempts, exp.nsamples)


def test_cli_interdict_byte_stable(host, golden, tmp_path):
    """proj/tests/test_cli.cpp:242-251: interdict --seed 42 --workers 1 --omit-timing is byte-stable
    against tests/golden/interdict12.json."""
    fx = golden["fixture12_given"]
    w = _hexlist(fx["weight"])
    edges = tmp_path / "fixture12.edges"
    edges.write_text("".join(f"{fx['in_src'][e]} {fx['edge_dst'][e]} {float(w[e])!r}\n"
                             for e in range(fx["m"])))
    sus = tmp_path / "fixture12.suspects"
    sus.write_text("2 1.0\n5 0.8\n9 0.6\n")
    out = tmp_path / "out.json"
    rc = host.run_cli(["interdict", "--graph", str(edges), "--weights", "given", "--suspects",
                       str(sus), "--mode", "edge", "--k", "3", "--epsilon", "0.3", "--delta", "0.2",
                       "--seed", "42", "--workers", "1", "--omit-timing", "--output", str(out)])
    assert rc == 0
    assert out.read_text() == fx["interdict12_json_text"]
    rc = host.run_cli(["sample", "--graph", str(edges), "--weights", "given", "--suspects", str(sus),
                       "--target", "200", "--seed", "42", "--output", str(out), "--dump",
                       str(tmp_path / "walks.txt")])
    assert rc == 0
    j = json.loads(out.read_text())
    exp = fx["pool_seed42_target200"]
    assert j["accepted"] == exp["nsamples"] and j["attempts"] == exp["attempts"]
    lines = (tmp_path / "walks.txt").read_text().splitlines()
    assert len(lines) == exp["nsamples"]
    first = [int(x) for x in lines[0].split()]
    assert first[0] == exp["tag_worker"][0] and first[2] + 1 == len(first) - 3
    rc = host.run_cli(["interdict", "--graph", str(edges), "--weights", "given", "--suspects",
                       str(sus), "--k", "3", "--max-attempts", "50"])
    assert rc == 3  # SamplingError -> runtime error


@pytest.mark.parametrize("kind,k", [(0, 20), (1, 10)])
def test_bound_skip_does_not_change_results(host, synth3000, monkeypatch, kind, k):
    """Iterations whose R'_t cannot reach Lambda_1 skip greedy (solver.cpp): same InterdictionResult
    as running every iteration in full, as the reference does (interdiction.cpp:36-47)."""
    g = host.Graph.from_csr(synth3000.n, synth3000.m, synth3000.in_offsets, synth3000.in_src,
                            synth3000.in_cum)
    monkeypatch.setenv("HSAW_SKIP_BOUND", "0")
    full = host.interdict(g, synth3000.p_of, kind, k, 0.1, 0.05, seed=5)
    monkeypatch.delenv("HSAW_SKIP_BOUND")
    fast = host.interdict(g, synth3000.p_of, kind, k, 0.1, 0.05, seed=5)
    assert full == fast and full["iterations"] >= 2


@pytest.mark.parametrize("kind,k", [(0, 20), (1, 10)])
def test_greedy_coverage_is_the_in_sample_coverage(host, synth3000, monkeypatch, kind, k):
    """The doubling loop takes Cov_R(S) from the greedy run (the walks of a stream are
    self-avoiding, so the sum of the marginal gains is the number of walks S covers) instead of a
    second coverage_of pass over R_t; HSAW_RECOUNT_COVERAGE=1 runs that pass as the reference does
    (coverage.cpp:212-231). Same InterdictionResult either way."""
    g = host.Graph.from_csr(synth3000.n, synth3000.m, synth3000.in_offsets, synth3000.in_src,
                            synth3000.in_cum)
    monkeypatch.setenv("HSAW_RECOUNT_COVERAGE", "1")
    recounted = host.interdict(g, synth3000.p_of, kind, k, 0.1, 0.05, seed=5)
    monkeypatch.delenv("HSAW_RECOUNT_COVERAGE")
    fast = host.interdict(g, synth3000.p_of, kind, k, 0.1, 0.05, seed=5)
    assert recounted == fast and fast["iterations"] >= 2

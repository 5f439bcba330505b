"""Ranking baselines, CPU side: the oracle restatement (orc_rr_node_sets +
oracle.Port.baseline) and the host layer's score rankings against the unmodified reference's
baseline() outputs (tests/golden/make_baseline_golden.py). Mirrors
proj/tests/test_evaluation.cpp:165-246."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR
from oracle.oracle import BuildError
from test_partition_cpu import host, pcsr, pv  # noqa: F401


@pytest.fixture(scope="module")
def bv():
    with open(os.path.join(GOLDEN_DIR, "baseline_vectors.json")) as f:
        return json.load(f)


def shim_weights(csr):
    """ProbGraph::weight as ref_graph_from_csr / hsaw::graph_from_csr derive it: in_cum differences."""
    off = csr.in_offsets.astype(np.int64)
    prev = np.concatenate([[0.0], csr.in_cum[:-1]])
    prev[off[:-1][np.diff(off) > 0]] = 0.0
    return csr.in_cum - prev


def test_oracle_baselines_match_reference(bv, pcsr, port):  # noqa: F811
    w = shim_weights(pcsr)
    for c in bv["cases"]:
        if "error" in c:
            with pytest.raises(BuildError):
                port.baseline(pcsr, w, c["kind"], c["mode"], c["k"], bv["state0"], bv["infmax_samples"])
            continue
        ids, s = port.baseline(pcsr, w, c["kind"], c["mode"], c["k"], bv["state0"],
                               bv["infmax_samples"])
        assert [int(x) for x in ids] == c["ids"] and s == c["state"], c


def test_rr_sets_are_simple_reverse_walks(pcsr, port):  # noqa: F811
    """evaluation.cpp:169-191: every set is a reverse walk without repeats, and it stops only at a
    dead end or a repeat (1 + |set| draws each, so the state after pins the lengths)."""
    s0 = port.seed_from_worker(4)
    off, items, s1 = port.rr_node_sets(pcsr, s0, 500)
    assert off[0] == 0 and off[-1] == items.size
    dst = np.repeat(np.arange(pcsr.n), np.diff(pcsr.in_offsets).astype(np.int64))
    edges = set(zip(pcsr.in_src.tolist(), dst.tolist()))
    for i in range(500):
        nodes = items[int(off[i]):int(off[i + 1])].tolist()
        assert len(set(nodes)) == len(nodes) >= 1
        assert all((nodes[j + 1], nodes[j]) in edges for j in range(len(nodes) - 1))
    s = s0
    for _ in range(int(off[-1]) + 500):
        s, _ = port.prg_next(s)
    assert s == s1


def test_host_score_rankings_match_reference(host, bv, pcsr):  # noqa: F811
    """Pagerank / MaxDegree / Randomized are host code (no device needed)."""
    g = host.Graph.from_csr(pcsr.n, pcsr.m, pcsr.in_offsets, pcsr.in_src, pcsr.in_cum)
    for c in bv["cases"]:
        if c["kind"].startswith("infmax"):
            continue
        if "error" in c:
            with pytest.raises(host.HsawError):
                host.baseline(g, pcsr.p_of, c["kind"], c["mode"], c["k"], bv["state0"])
            continue
        ids, s = host.baseline(g, pcsr.p_of, c["kind"], c["mode"], c["k"], bv["state0"])
        assert ids == c["ids"] and s == c["state"], c

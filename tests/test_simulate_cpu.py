"""CPU side of the paired LT forward simulation: the oracle restatement of
proj/src/evaluation.cpp:49-108,195-242 against the reference-generated goldens
(tests/golden/evaluation_vectors.json, made by make_eval_golden.py), against the reference's own
test cases (proj/tests/test_evaluation.cpp:13-78) and, where oracle/_ref is present, against the
compiled reference live. The device path is covered by tests/test_gpu_simulate.py."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR
from oracle.oracle import Csr, OracleError

BUDGET = 5e7  # draws the CPU suite is willing to replay per case


@pytest.fixture(scope="module")
def eval_golden():
    with open(os.path.join(GOLDEN_DIR, "evaluation_vectors.json")) as f:
        return json.load(f)


def _graphs(fixture12, fixture12_indegree, synth3000):
    return {"fixture12_given": fixture12, "config1_indegree": fixture12_indegree,
            "synth3000": synth3000}


def two_node():  # proj/tests/oracles.hpp:130-137
    return Csr(2, 1, np.array([0, 1, 1], dtype=np.uint64), np.array([1], dtype=np.uint32),
               np.array([0.5]), np.array([0.0, 1.0]))


def test_oracle_matches_reference_goldens(port, eval_golden, fixture12, fixture12_indegree,
                                          synth3000):
    checked = 0
    for name, csr in _graphs(fixture12, fixture12_indegree, synth3000).items():
        g = eval_golden[name]
        f = g["lt_forward_simulate"]
        s, got = f["state0"], []
        for _ in f["infected"]:
            cnt, s = port.lt_forward_simulate(csr, s)
            got.append(cnt)
        assert got == f["infected"] and s == f["state_after"]
        members = int(np.count_nonzero(csr.p_of))
        for c in g["estimate_suspension"]:
            if c["runs"] * (csr.n + members) > BUDGET:
                continue
            e = port.estimate_suspension(csr, c["kind"], c["ids"], c["epsilon"], c["delta"],
                                         c["state0"])
            assert e == dict(value=float.fromhex(c["value"]), capped=c["capped"], runs=c["runs"],
                             state=c["state_after"]), (name, c["kind"], c["ids"][:4])
            checked += 1
    assert checked >= 20


def test_reference_forward_simulation_cases(port):  # test_evaluation.cpp:13-38
    chain = Csr(3, 2, np.array([0, 0, 1, 2], dtype=np.uint64), np.array([0, 1], dtype=np.uint32),
                np.array([1.0, 1.0]), np.array([1.0, 0.0, 0.0]))
    s = 3
    for _ in range(100):
        cnt, s = port.lt_forward_simulate(chain, s)
        assert cnt == 3
    full, _, _ = port.paired_runs(two_node(), 0, [], 11, 200000)
    assert abs(full.mean() - 1.5) < 0.0075  # "two-node mean tends to 1.5"


def test_reference_estimator_cases(port):  # test_evaluation.cpp:40-66
    g = two_node()
    e = port.estimate_suspension(g, 0, [], 0.1, 0.1, 21)
    assert e["value"] == 0.0 and not e["capped"] and e["state"] == 21
    e = port.estimate_suspension(g, 0, [0], 0.05, 0.05, 21)
    assert abs(e["value"] - 0.5) / 0.5 < 0.05
    e = port.estimate_suspension(g, 1, [1], 0.05, 0.05, 21)
    assert abs(e["value"] - 1.5) / 1.5 < 0.05
    for eps, delta in ((0.0, 0.1), (0.1, 1.0)):
        with pytest.raises(OracleError) as ei:
            port.estimate_suspension(g, 0, [0], eps, delta, 21)
        assert ei.value.status == 1
    with pytest.raises(OracleError) as ei:
        port.estimate_suspension(g, 0, [1], 0.1, 0.1, 21)
    assert ei.value.status == 2


def test_oracle_equals_reference_live(port, ref):
    from paper_1702_05854_b200 import rmat
    for seed in (3, 4):
        r = rmat.rmat_graph(10, 8.0, seed=seed, suspect_frac=0.03, suspect_seed=seed + 1)
        csr = Csr(r.n, r.m, r.in_offsets, r.in_src, r.in_cum, r.p_of)
        rng = np.random.Generator(np.random.PCG64(seed))
        with ref.handles(csr) as hd:
            s0 = port.seed_from_worker(seed)
            a, b = s0, s0
            for _ in range(4):
                ca, a = port.lt_forward_simulate(csr, a)
                cb, b = ref.lt_forward_simulate(csr, b, hd=hd)
                assert (ca, a) == (cb, b)
            for kind in (0, 1):
                limit = csr.m if kind == 0 else csr.n
                ids = np.unique(rng.integers(0, limit, size=limit // 10))
                assert port.estimate_suspension(csr, kind, ids, 0.3, 0.2, s0) == \
                    ref.estimate_suspension(csr, kind, ids, 0.3, 0.2, s0, hd=hd)


def test_host_layer_argument_checks_without_a_device():
    """hsaw::estimate_suspension(g, vi, ...) checks its arguments in the reference's order before
    touching the device (evaluation.cpp:214-218), and fails loudly — no CPU fallback — after."""
    import torch
    from paper_1702_05854_b200 import hostapi
    g = hostapi.Graph.synth(50, 3, 1)
    p_of = g.random_suspects(5, seed=2)
    for eps, delta, status in ((0.0, 0.1, 1), (0.5, 1.0, 1)):
        with pytest.raises(hostapi.HsawError) as ei:
            hostapi.estimate_suspension(g, p_of, 0, [0], eps, delta, 1)
        assert ei.value.status == status
    with pytest.raises(hostapi.HsawError) as ei:
        hostapi.estimate_suspension(g, p_of, 0, [g.m], 0.3, 0.2, 1)
    assert ei.value.status == 2 and "removal id out of range" in str(ei.value)
    assert hostapi.estimate_suspension(g, p_of, 1, [], 0.3, 0.2, 77) == \
        dict(value=0.0, capped=False, runs=0, state=77)
    if not torch.cuda.is_available():
        with pytest.raises(hostapi.HsawError) as ei:
            hostapi.estimate_suspension(g, p_of, 0, [0], 0.3, 0.2, 1)
        assert ei.value.status == 5  # DeviceError

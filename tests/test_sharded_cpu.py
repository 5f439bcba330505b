"""Multi-rank orchestration on CPU: world_size 2 over gloo (127.0.0.1), each rank driving a
test-side engine (tests/cpu_engine.py). The sharded solver must reproduce the single-stream
results — same R_t / R'_t cut, solution, coverage, attempts, est_suspension — for every world size
(SURVEY.md §8b "determinism contract": identical across GPU counts)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN_DIR, ROOT


def test_layout_bookkeeping():
    from paper_1702_05854_b200.sharded import Layout, Round
    assert Layout.split(0, 10, 4) == [3, 3, 2, 2]
    assert Layout.split(0, 2, 4) == [1, 1, 0, 0]
    lay = Layout(2, [Round(0, [3, 2], [5, 1]), Round(5, [2, 2], [0, 4]), Round(9, [1, 0], [2, 0])])
    assert (lay.accepted, lay.batches) == (12, 10)
    # global order: r0:[0,5) r1:[5,6) | r0:[] r1:[6,10) | r0:[10,12)
    assert lay.local_range(0, 0, 12) == (0, 7) and lay.local_range(1, 0, 12) == (0, 5)
    assert lay.local_range(0, 0, 6) == (0, 5) and lay.local_range(1, 0, 6) == (0, 1)
    assert lay.local_range(0, 6, 6) == (5, 2) and lay.local_range(1, 6, 6) == (1, 4)
    assert lay.local_range(0, 3, 4) == (3, 2) and lay.local_range(1, 3, 4) == (0, 2)
    assert lay.locate(5) == (0, 0, 0) and lay.locate(6) == (0, 1, 5)
    assert lay.locate(7) == (1, 1, 6) and lay.locate(12) == (2, 0, 10) and lay.locate(13) is None
    for r in range(2):  # ranges tile the local storage without gaps for consecutive global slices
        a = lay.local_range(r, 0, 4)
        b = lay.local_range(r, 4, 8)
        assert a[0] + a[1] == b[0]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_no, case, out_q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import json

    import torch.distributed as dist

    from cpu_engine import CpuEngine
    from oracle.oracle import Csr, Port
    from paper_1702_05854_b200.sharded import Comm, ShardedSolver

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        with open(os.path.join(GOLDEN_DIR, "reference_vectors.json")) as f:
            golden = json.load(f)
        hx = lambda xs: np.array([float.fromhex(x) for x in xs])
        fx = golden["fixture12_given"]
        if case["graph"] == "fixture12":
            csr = Csr(fx["n"], fx["m"], np.array(fx["in_offsets"], dtype=np.uint64),
                      np.array(fx["in_src"], dtype=np.uint32), hx(fx["in_cum"]), hx(fx["p_of"]))
        elif case["graph"] == "config1":
            c1 = golden["config1_indegree"]["seed42"]
            csr = Csr(fx["n"], fx["m"], np.array(fx["in_offsets"], dtype=np.uint64),
                      np.array(fx["in_src"], dtype=np.uint32), hx(c1["in_cum"]), hx(c1["p_of"]))
        else:
            z = np.load(os.path.join(GOLDEN_DIR, "synth3000.npz"))
            csr = Csr(z["in_offsets"].size - 1, z["in_src"].size, z["in_offsets"], z["in_src"],
                      z["in_cum"], z["p_of"])
        eng = CpuEngine(Port(), csr, case["seed"], max_attempts=case.get("max_attempts", 10**8))
        solver = ShardedSolver(eng, Comm())
        if case.get("expect_budget"):
            try:
                solver.ensure(case["target"])
                res = "no error"
            except Exception as e:  # noqa: BLE001
                res = getattr(e, "status", repr(e))
        elif "removal" in case:
            members = int(np.count_nonzero(csr.p_of))
            res = solver.estimate_suspension(csr.n, members, case["kind"], case["removal"],
                                             case["eps"], case["delta"], case["state"],
                                             batch_runs=case.get("batch_runs"))
        elif "target" in case:
            solver.ensure(case["target"])
            res = dict(counters=solver.counters_for(case["target"]),
                       accepted=solver.layout.accepted, local=solver.local_accepted)
        else:
            res = solver.interdict(csr.n, case["kind"], case["k"], case["eps"], case["delta"],
                                   cand=case.get("cand"))
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


def run_case(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_no, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


def test_sharded_esia_matches_reference_golden(golden):
    fx = golden["fixture12_given"]
    res = run_case(dict(graph="fixture12", seed=42, kind=0, k=3, eps=0.3, delta=0.2))
    assert res[0] == res[1] == fx["interdict_edge_k3"]
    c = fx["interdict_edge_k3_cand"]
    res = run_case(dict(graph="fixture12", seed=7, kind=0, k=3, eps=0.3, delta=0.2, cand=c["cand"]))
    assert res[0] == res[1] == c["result"]


def test_sharded_nsia_config1_three_ranks(golden):
    c1 = golden["config1_indegree"]["seed42"]
    res = run_case(dict(graph="config1", seed=42, kind=1, k=5, eps=0.1, delta=0.1), world=3)
    assert res[0] == res[1] == res[2] == c1["nsia_k5"]


def test_sharded_counters_and_budget(golden, port, synth3000):
    exp = golden["synth3000"]["pool_seed5_target4000"]
    res = run_case(dict(graph="synth3000", seed=5, target=4000))
    assert res[0]["counters"] == res[1]["counters"] == (exp["attempts"], exp["nsamples"])
    assert res[0]["accepted"] == res[1]["accepted"] == res[0]["local"] + res[1]["local"]
    res = run_case(dict(graph="fixture12", seed=1, target=10**6, max_attempts=3000,
                        expect_budget=True))
    assert res[0] == res[1] == 3  # SamplingError on every rank


def test_prg_jump_equals_stepping(port):
    """capi.prg_jump (GF(2) jump-ahead of xorshift64*, host arithmetic of the C-ABI library)."""
    from paper_1702_05854_b200 import capi
    s = port.seed_from_worker(3)
    x = s
    for i in range(1, 200):
        x, _ = port.prg_next(x)
        assert capi.prg_jump(s, i) == x
    assert capi.prg_jump(s, 0) == s
    a = capi.prg_jump(s, 10**12 + 7)
    assert capi.prg_jump(capi.prg_jump(s, 10**12), 7) == a


def test_sharded_estimate_suspension_matches_reference_golden():
    import json
    with open(os.path.join(GOLDEN_DIR, "evaluation_vectors.json")) as f:
        ev = json.load(f)
    # synth3000, edge removal, eps 0.3: 4024 runs in the reference
    c = ev["synth3000"]["estimate_suspension"][0]
    want = dict(value=float.fromhex(c["value"]), capped=c["capped"], runs=c["runs"],
                state=c["state_after"])
    res = run_case(dict(graph="synth3000", seed=0, kind=c["kind"], removal=c["ids"],
                        eps=c["epsilon"], delta=c["delta"], state=c["state0"], batch_runs=1000))
    assert res[0] == res[1] == want
    # fixture12 node removal on three ranks, small uneven batches
    c = ev["fixture12_given"]["estimate_suspension"][3]
    want = dict(value=float.fromhex(c["value"]), capped=c["capped"], runs=c["runs"],
                state=c["state_after"])
    res = run_case(dict(graph="fixture12", seed=0, kind=c["kind"], removal=c["ids"],
                        eps=c["epsilon"], delta=c["delta"], state=c["state0"], batch_runs=101),
                   world=3)
    assert res[0] == res[1] == res[2] == want

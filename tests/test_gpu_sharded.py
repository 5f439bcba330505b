"""Sharded solver on the real kernels. One GPU is available, so: world 1 through the sharded code
path, and world 2 as two processes sharing cuda:0 with gloo carrying the (tiny) collectives through
the host — the device-side steps (sample_range, rounds begin/select/cover/apply, coverage) are the
production ones; only the transport differs from NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN_DIR, ROOT, upload

pytestmark = pytest.mark.gpu


def test_world1_equals_single_gpu_path(ctx, gpu_lib, golden, synth3000):
    from paper_1702_05854_b200.sharded import GpuEngine, ShardedSolver
    upload(ctx, synth3000)
    for kind, key in ((0, "esia_k5"), (1, "nsia_k5")):
        eng = GpuEngine(ctx, seed=3)
        try:
            res = ShardedSolver(eng).interdict(synth3000.n, kind, 5, 0.2, 0.1)
        finally:
            eng.close()
        assert res == golden["synth3000"][key]


def test_world1_estimate_suspension_equals_reference_golden(ctx, synth3000):
    """ShardedSolver.estimate_suspension on the device engine: run ranges addressed by stream
    position (capi.prg_jump) give the reference's value / runs / state."""
    import json
    from paper_1702_05854_b200.sharded import GpuEngine, ShardedSolver
    with open(os.path.join(GOLDEN_DIR, "evaluation_vectors.json")) as f:
        cases = json.load(f)["synth3000"]["estimate_suspension"]
    upload(ctx, synth3000)
    members = int(np.count_nonzero(synth3000.p_of))
    eng = GpuEngine(ctx, seed=0)
    try:
        for c in cases[:4]:
            got = ShardedSolver(eng).estimate_suspension(synth3000.n, members, c["kind"], c["ids"],
                                                         c["epsilon"], c["delta"], c["state0"],
                                                         batch_runs=777)
            assert got == dict(value=float.fromhex(c["value"]), capped=c["capped"],
                               runs=c["runs"], state=c["state_after"])
    finally:
        eng.close()


def test_rounds_session_matches_fused_greedy(ctx, gpu_lib, synth3000):
    """The stepwise rounds API alone (one rank) equals hsaw_gpu_greedy."""
    import torch
    upload(ctx, synth3000)
    with ctx.stream(seed=8) as st:
        st.ensure(5000)
        for kind, limit in ((0, synth3000.m), (1, synth3000.n)):
            exp_sol, exp_cov = ctx.greedy(25, stream=st, kind=kind, off=0, cnt=5000)
            counts = torch.zeros(limit + 4, dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()
            r = gpu_lib.Rounds(ctx, counts.data_ptr(), stream=st, kind=kind, off=0, cnt=5000)
            lst = torch.empty(max(r.occurrences, 1), dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()
            sol, cov, replay = [], 0, []
            for _ in range(25):
                item, gain = r.select()
                sol.append(item)
                cov += gain
                n = r.cover(item, lst.data_ptr(), lst.numel())
                replay.append(lst[:n].clone())
            r.close()
            assert sol == exp_sol.tolist() and cov == exp_cov
            # replaying the decrement lists on a fresh histogram reproduces the final counts
            fresh = torch.zeros(limit + 4, dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()
            r2 = gpu_lib.Rounds(ctx, fresh.data_ptr(), stream=st, kind=kind, off=0, cnt=5000)
            for items in replay:
                r2.apply(items.data_ptr(), items.numel())
            ctx.sync()
            r2.close()
            assert torch.equal(fresh, counts)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_no, kind, k, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1702_05854_b200 import capi
    from paper_1702_05854_b200.sharded import Comm, GpuEngine, ShardedSolver

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z = np.load(os.path.join(GOLDEN_DIR, "synth3000.npz"))
        n, m = z["in_offsets"].size - 1, z["in_src"].size
        with capi.Context(0) as ctx:
            ctx.upload_graph(n, m, z["in_offsets"], z["in_src"], z["in_cum"], z["p_of"])
            eng = GpuEngine(ctx, seed=3)
            try:
                if isinstance(kind, dict):  # a forward-simulation case (estimate_suspension)
                    c = kind
                    res = ShardedSolver(eng, Comm()).estimate_suspension(
                        n, int(np.count_nonzero(z["p_of"])), c["kind"], c["ids"], c["epsilon"],
                        c["delta"], c["state0"], batch_runs=513)
                else:
                    res = ShardedSolver(eng, Comm()).interdict(n, kind, k, 0.2, 0.1)
            finally:
                eng.close()
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,key", [(0, "esia_k5"), (1, "nsia_k5")])
def test_two_ranks_on_one_gpu(golden, kind, key):
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port_no = _free_port()
    procs = [mpc.Process(target=_worker, args=(r, 2, port_no, kind, 5, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[0] == results[1] == golden["synth3000"][key]


def test_two_ranks_on_one_gpu_estimate_suspension():
    """Runs of the paired forward simulation split over two processes (device kernels on cuda:0,
    gloo for the per-batch all-gather of the counts): the reference's value / runs / state."""
    import json
    with open(os.path.join(GOLDEN_DIR, "evaluation_vectors.json")) as f:
        c = json.load(f)["synth3000"]["estimate_suspension"][2]
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port_no = _free_port()
    procs = [mpc.Process(target=_worker, args=(r, 2, port_no, c, 0, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = dict(value=float.fromhex(c["value"]), capped=c["capped"], runs=c["runs"],
                state=c["state_after"])
    assert results[0] == results[1] == want


def test_gathered_greedy_with_threshold_and_fallback(gpu_lib):
    """The gather-and-replicate greedy of the sharded solve on an instance large enough for a
    threshold above 1 (R-MAT 2^16, ~4e5 walks, > 2^20 items): the reduced walk set selects what the
    single-GPU greedy selects, the sharded upper bound equals the single-GPU one, and a budget deep
    into the low counts (k-th gain below the threshold) takes the full-gather fallback."""
    import torch
    from paper_1702_05854_b200 import hostapi
    from paper_1702_05854_b200.sharded import GpuEngine, ShardedSolver
    g = hostapi.Graph.rmat(16, 16.0, seed=1)
    p_of = g.random_suspects(g.n // 100, seed=2)
    with hostapi.DeviceGraph(g, p_of) as dg:
        ctx = gpu_lib.Context.borrow(dg.ctx_handle(), g.n, g.m)
        eng = GpuEngine(ctx, seed=42, cfg=gpu_lib.SamplerCfg(max_attempts=10**12))
        try:
            solver = ShardedSolver(eng)
            solver.ensure(400_000)
            for kind in (0, 1):
                counts = eng.local_counts(kind, 0, 200_000, None)
                mc = eng.threshold_from_counts(counts)
                assert mc > 1
                lens, items = eng.reduced_walks(kind, 0, 200_000, counts, mc)
                c = counts.cpu().numpy()
                it = items.cpu().numpy()
                assert lens.sum().item() == items.numel() and np.all(c[it] >= mc)
                assert items.numel() == int(c[c >= mc].sum())  # every occurrence of an indexed item
                # counts handed over at any alignment (a view that starts 4 bytes into the buffer)
                assert eng.bound_from_counts(counts[1:], 100, 10**12) == \
                    eng.bound_from_counts(counts[1:].clone(), 100, 10**12)
                for k in (30, 3000):
                    exp_sol, exp_cov = ctx.greedy(k, stream=eng.stream, kind=kind, off=0, cnt=200_000)
                    sol, cov = solver.greedy(k, kind, 200_000)
                    assert sol == exp_sol.tolist() and cov == exp_cov
                exp_b = ctx.coverage_upper_bound(100, stream=eng.stream, kind=kind, off=200_000,
                                                 cnt=200_000)
                assert solver.coverage_upper_bound(100, kind, 200_000, 200_000) == exp_b
        finally:
            eng.close()
        res = hostapi.interdict(g, p_of, 0, 50, 0.1, 1.0 / g.n, seed=42, max_attempts=10**12, dg=dg)
        eng = GpuEngine(ctx, seed=42, cfg=gpu_lib.SamplerCfg(max_attempts=10**12))
        try:
            got = ShardedSolver(eng).interdict(g.n, 0, 50, 0.1, 1.0 / g.n)
        finally:
            eng.close()
        assert got == res


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
def test_cpp_multi_device_solve_equals_single_device(golden, synth3000, devices):
    """The C++ multi-device solve (host/multi.cpp, InterdictionOptions::devices) with 2 and 3 ranks
    sharing cuda:0: rank threads, sharded ensure / counters / coverage / bound, gather-and-replicate
    greedy over the in-process exchange — the reference's golden results, bit for bit."""
    from paper_1702_05854_b200 import hostapi
    g = hostapi.Graph.from_csr(synth3000.n, synth3000.m, synth3000.in_offsets, synth3000.in_src,
                               synth3000.in_cum)
    for kind, key in ((0, "esia_k5"), (1, "nsia_k5")):
        res = hostapi.interdict_devices(g, synth3000.p_of, kind, 5, 0.2, 0.1, devices, seed=3)
        assert res == golden["synth3000"][key]


def test_cpp_multi_device_solve_at_scale_16(tmp_path):
    """A larger instance (threshold > 1 in the gathered greedy, several sampling rounds) and the
    CLI flag: `hsaw interdict --devices 0,0` prints the single-device document."""
    import json
    from paper_1702_05854_b200 import hostapi
    g = hostapi.Graph.rmat(16, 16.0, seed=1)
    p_of = g.random_suspects(g.n // 100, seed=2)
    one = hostapi.interdict(g, p_of, 0, 50, 0.1, 1.0 / g.n, seed=42, max_attempts=10**12)
    two = hostapi.interdict_devices(g, p_of, 0, 50, 0.1, 1.0 / g.n, [0, 0], seed=42,
                                    max_attempts=10**12)
    assert two == one
    n1 = hostapi.interdict(g, p_of, 1, 20, 0.1, 1.0 / g.n, seed=7, max_attempts=10**12)
    n3 = hostapi.interdict_devices(g, p_of, 1, 20, 0.1, 1.0 / g.n, [0, 0, 0], seed=7,
                                   max_attempts=10**12)
    assert n3 == n1
    cache, sus = tmp_path / "g.hsaw1", tmp_path / "s.txt"
    small = hostapi.Graph.synth(2000, 6, 3)
    small.save_cache(cache)
    sp = small.random_suspects(40, 2)
    sus.write_text("".join(f"{v} {float(sp[v])!r}\n" for v in np.nonzero(sp)[0]))
    outs = []
    for extra in ([], ["--devices", "0,0"]):
        out = tmp_path / f"o{len(outs)}.json"
        rc = hostapi.run_cli(["interdict", "--graph", str(cache), "--suspects", str(sus), "--k", "4",
                              "--seed", "5", "--omit-timing", "--output", str(out)] + extra)
        assert rc == 0
        outs.append(json.loads(out.read_text()))
    assert outs[0] == outs[1]

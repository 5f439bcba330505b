#!/usr/bin/env python
"""bench.py — HSAWs/sec (and eSIA seconds-to-solution) of the B200 HSAW path.

Contract: `python bench.py --gpus N --steps K --warmup W [--impl reference]` prints ONE JSON line.

Workload at N=1 = BASELINE.json configs[1] ("C2"): R-MAT scale 20 (2^20 nodes, ~16.1 M edges after
dedupe), LT weights 1/in-degree, 1 % suspects with p ~ U(0,1), stream seed 42, the reference's
default sampler (Brent + window 2, 10 chained attempts per batch).
A *step* = one pass of the sampling hot path over one batch range: 2^20 batches (10.49 M attempts)
are generated (K1), replayed (K2), exactly rechecked (K2b) and compacted into the device-resident
pool in the reference's (batch, seq) order. `value` = accepted (post-recheck) HSAWs per second over
the K timed steps with the graph already resident in HBM. `e2e` = the same metric through the
reference-facing host call with HOST buffers (graph arrays uploaded inside the timed region, result
counters read back). The eSIA k=100 seconds-to-solution of the same config rides along in "esia".
With --gpus N>1 (torchrun) the graph is replicated, every rank samples its own batch ranges (weak
scaling, no data-path collective) and the rates are summed over ranks / max over ranks' time.

--impl reference times the reference's own CPU implementation (oracle/_ref: the unmodified
/root/reference sources compiled by oracle/Makefile; the C restatement if that is absent) on the
host cores with all hardware threads, on the same graph, metric and unit.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "hsaw_per_sec"
UNIT = "HSAW/s"
STREAM_SEED = 42


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scale", type=int, default=20, help="R-MAT scale (2^scale nodes)")
    ap.add_argument("--edge-factor", type=float, default=16.0)
    ap.add_argument("--batches", type=int, default=1 << 20, help="batches per step per GPU")
    ap.add_argument("--esia-k", type=int, default=100)
    ap.add_argument("--no-esia", action="store_true")
    ap.add_argument("--solver", default="esia", choices=["esia", "nsia"],
                    help="interdiction driver timed beside the sampler (edge or node candidates)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ingest", action="store_true",
                    help="also time the step before the path (SURVEY 8f row 1): HSAW1 cache and "
                         "edge-list text of a graph of this size -> ProbGraph / resident graph, "
                         "device loaders vs the host loaders, the reference's loaders as cpu_baseline")
    ap.add_argument("--no-suspension", action="store_true",
                    help="skip the forward-simulation leg (estimate_suspension of the solution)")
    ap.add_argument("--no-l2-flush", action="store_true",
                    help="A/B only: skip the L2 flush between timed steps")
    ap.add_argument("--cpu-target", type=int, default=300_000,
                    help="HSAWs of the bounded CPU sample (cpu_baseline / reference arm step)")
    return ap.parse_args()


def workload_name(args, n, m):
    return (f"C2 R-MAT scale {args.scale} ({n} nodes, {m} edges after dedupe), LT weights "
            f"1/in-degree, {max(1, n // 100)} suspects p~U(0,1), stream seed {STREAM_SEED}, "
            f"Brent+window(2), 10 attempts/batch")


def make_inputs(args):
    """The same CSR arrays go to the GPU path and to the CPU reference."""
    from paper_1702_05854_b200 import hostapi
    g = hostapi.Graph.rmat(args.scale, args.edge_factor, seed=1)
    p_of = g.random_suspects(max(1, g.n // 100), seed=2)
    return g, p_of


class ClockSampler(threading.Thread):
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        super().__init__(daemon=True)
        self.index, self.rows, self._halt = index, [], threading.Event()

    def run(self):
        while not self._halt.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._halt.wait(0.2)

    def stop(self) -> dict:
        self._halt.set()
        self.join(timeout=6)
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows if len(r) >= 8
                          for n, v in zip(names, r[4:8]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md, 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per K1 launch from the committed ncu capture, if one exists for this workload."""
    try:
        with open(os.path.join(ROOT, "profiles", "k1_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


def cpu_reference_rate(args, g, p_of, target, seed, workers):
    """Reference CPU stream_samples on the host cores -> (HSAW/s, accepted, attempts, kind)."""
    from oracle import oracle
    from oracle.oracle import Csr
    off, src, cum, _, _ = g.arrays()
    csr = Csr(g.n, g.m, off, src, cum, p_of)
    if oracle.have_ref():
        R = oracle.Ref()
        with R.handles(csr) as hd:
            t0 = time.perf_counter()
            ns, at, _ = R.stream_samples(csr, target, seed=seed, workers=workers,
                                         max_attempts=10**12, hd=hd, copy=False)
            dt = time.perf_counter() - t0
        return ns / dt, ns, at, "reference", workers, dt
    P = oracle.Port()
    t0 = time.perf_counter()
    pool = P.stream_samples(csr, target, seed=seed, max_attempts=10**12)
    dt = time.perf_counter() - t0
    return pool.nsamples / dt, pool.nsamples, pool.attempts, "port", 1, dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    g, p_of = make_inputs(args)
    cores = os.cpu_count() or 1
    total, elapsed, kind, used = 0, 0.0, "reference", cores
    for step in range(args.warmup + args.steps):
        rate, ns, at, kind, used, dt = cpu_reference_rate(args, g, p_of, args.cpu_target,
                                                          STREAM_SEED + step, cores)
        if step >= args.warmup:
            total += ns
            elapsed += dt
    value = total / elapsed if elapsed > 0 else 0.0
    sample = (f"each step: stream_samples to {args.cpu_target} HSAWs (fresh stream seed "
              f"{STREAM_SEED}+step) with {used} worker threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * elapsed / max(args.steps, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64/f64", "data": "synthetic",
        "config": {"workload": workload_name(args, g.n, g.m), "step": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }))


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_1702_05854_b200 import capi, hostapi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device — the HSAW path has no CPU fallback")
    # Test hook (one-GPU boxes): HSAW_BENCH_ONE_GPU=1 puts every rank on cuda:0 and swaps NCCL for
    # gloo, so the N > 1 control flow can be exercised where only one device exists.
    one_gpu = os.environ.get("HSAW_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def all_reduce(t, op):
        if one_gpu:  # gloo reduces host tensors
            h = t.cpu()
            dist.all_reduce(h, op=op)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op)

    g, p_of = make_inputs(args)  # identical on every rank (seeded generator): replicated graph
    off, src, cum, _, _ = g.arrays()
    ref_bytes = 8 * (g.n + 1) + 12 * g.m + 8 * g.n

    tstream = torch.cuda.Stream()
    dg = hostapi.DeviceGraph(g, p_of, device=local, cuda_stream=tstream.cuda_stream)
    ctx = capi.Context.borrow(dg.ctx_handle(), g.n, g.m)
    cfg = capi.SamplerCfg(max_attempts=10**15)
    B = args.batches

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    step_index = [0]
    replay_counts = []

    def one_step():
        # weak scaling: global batch ranges are dealt round-robin to the ranks; no collective on
        # the data path. Each step samples its range into a fresh SampleStream, so the walk pool
        # of the previous step is recycled instead of growing without bound over K steps.
        first = (step_index[0] * world + rank) * B
        step_index[0] += 1
        with ctx.stream(seed=STREAM_SEED, cfg=cfg) as st:
            got = st.sample_range(first, B)
            replay_counts.append(st.stats()["spare"])
        return got

    for _ in range(args.warmup):
        one_step()
    barrier()
    ctx.stage_times(reset=True)
    launches0 = ctx.launches
    first_timed_step = step_index[0]
    clocks = ClockSampler(local)
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    accepted = 0
    # L2 is flushed between timed steps by overwriting a buffer twice its size on the launching
    # stream, so every step starts with a cold L2 and re-reads the graph from HBM. Each step is
    # bracketed by its own event pair (the flush sits between the pairs: it is apparatus, not
    # workload); the outer bracket, flushes included, is reported next to it.
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    pairs = []
    with torch.cuda.stream(tstream):
        ev0.record(tstream)
        for _ in range(args.steps):
            if not args.no_l2_flush:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(tstream)
            accepted += one_step()
            b.record(tstream)
            pairs.append((a, b))
        ev1.record(tstream)
    barrier()
    outer_ms = ev0.elapsed_time(ev1)
    elapsed_ms = sum(a.elapsed_time(b) for a, b in pairs)
    clock_info = clocks.stop()
    stages = ctx.stage_times(reset=True)
    launches = ctx.launches - launches0
    # Algorithmic work of exactly the timed batch ranges, counted by an untimed instrumented pass
    # (the production kernels run with the counters compiled out).
    delta = {k: 0 for k in capi.STAT_NAMES}
    for st_i in range(first_timed_step, first_timed_step + args.steps):
        first = (st_i * world + rank) * B
        one = ctx.encode_stats(STREAM_SEED + first, B, cfg)
        for k in delta:
            delta[k] += one[k]

    t = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda")
    c = torch.tensor([accepted, delta["attempts"], delta["steps"], launches],
                     dtype=torch.float64, device="cuda")
    if world > 1:
        all_reduce(t, dist.ReduceOp.MAX)
        all_reduce(c, dist.ReduceOp.SUM)
    elapsed_ms = float(t.item())
    tot_acc, tot_att, tot_steps, tot_launches = (float(x) for x in c.tolist())
    value = tot_acc / (elapsed_ms / 1e3)

    # ---- roofline of the dominant kernel (K1 encode), rank 0's launches
    peak, peak_src = measured_peak()
    k1_ms, k1_n = stages["encode"]
    # K1 also materialises the accepted walks (8 B per walk item logged while walking); the
    # replay pass the reference needs for that (its K2) is not re-counted
    log_bytes = 8 * delta["spare"]
    alg_bytes_per_launch = (delta["alg_bytes"] + log_bytes) / max(k1_n, 1)
    k1_avg_ms = k1_ms / max(k1_n, 1)
    achieved = alg_bytes_per_launch / (k1_avg_ms / 1e3) / 1e9 if k1_avg_ms > 0 else 0.0
    traffic = ncu_traffic()
    # Secondary roofline in the kernel's own unit: random sector gathers. On the compact layout a
    # step is one in_src gather (live picks) plus one 16-byte header gather (arrivals, start nodes
    # included); tools/gather_probe.cu measured what this B200 sustains for dependent random
    # gathers (profiles/README.md): 212 G/s from a 64 MB table (L2 resident), 150 G/s at 96 MB,
    # 49 G/s from HBM (every miss costs a 128-byte line).
    gathers = (2 * delta["steps"] + delta["attempts"]) / max(k1_n, 1)
    roofline = {
        "bound": "hbm", "kernel": "encode_compact_kernel<Brent,2,record> (K1, walk generation + "
                                  "materialisation, compact L2-resident layout)",
        "achieved": achieved,
        "peak": peak, "unit": "GB/s", "frac": achieved / peak if peak else None,
        "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
        "peak_source": peak_src,
        "algorithmic_bytes_per_launch": alg_bytes_per_launch,
        "bytes_per_step_formula": "28+8*ceil(log2 d) per successful pick (16 empty row, 24 no "
                                  "live edge) + 8 per node arrival (SURVEY.md 8d) + 8 per item "
                                  "of an accepted walk (logged by the same kernel)",
        "note": "algorithmic bytes are the reference-layout figure of SURVEY.md 8(d); the device "
                "layout serves them from 4-byte sources + 16-byte row headers that stay in L2, so "
                "measured DRAM traffic (`traffic`) is a fraction of it and frac can exceed 1. The "
                "kernel's own limit is the random-gather rate below.",
        "walk_log_bytes_per_launch": log_bytes / max(k1_n, 1),
        "kernel_avg_ms": k1_avg_ms, "launches_timed": k1_n,
        "k1_walk_steps_per_s": delta["steps"] / (k1_ms / 1e3) if k1_ms > 0 else None,
        "gather": {"gathers_per_launch_upper": gathers,
                   "achieved_ggathers_per_s": gathers / (k1_avg_ms / 1e3) / 1e9 if k1_avg_ms else None,
                   "probe_peak_ggathers_per_s": {"l2_resident_64MB": 212.0, "96MB": 150.0,
                                                 "hbm_512MB": 49.0}},
        "stage_ms": {k: round(v[0], 3) for k, v in stages.items() if v[1]},
        "k1_share_of_step": k1_ms / elapsed_ms if elapsed_ms > 0 else None,
    }
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / max(args.steps, 1),
        "ms_per_step_incl_l2_flush": outer_ms / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64/f64",
        "data": "synthetic",
        "config": {
            "workload": workload_name(args, g.n, g.m),
            "step": f"{B} batches ({10 * B} attempts) per GPU: K1 encode+record, K2b exact recheck, "
                    f"ordered compaction into the device pool (K2 replay only on log overflow)",
            "layout": ("compact (in_src packed three 21-bit entries per 64-bit word + 16-byte row "
                       "headers, L2 resident)" if g.n <= 2**20 else
                       "compact (4-byte in_src + 16-byte row headers; headers L2 resident)")
                      if 16 * g.n <= 126 * 2**20 else "fat (32-byte edge records)",
            "parallelism": f"walks sharded by batch range over {world} GPU(s), graph replicated",
            "l2_policy": (f"L2 flushed before every timed step (256 MB memset on the launching "
                          f"stream between the per-step event pairs); graph on device "
                          f"{hsaw_mb(dg)} MB")
                         if not args.no_l2_flush else "NOT flushed (A/B run)",
            "graph_device_bytes": ctx.graph_bytes, "graph_reference_bytes": ref_bytes,
        },
        "attempts_per_sec": tot_att / (elapsed_ms / 1e3),
        "walk_steps_per_sec": tot_steps / (elapsed_ms / 1e3),
        "accept_rate": tot_acc / tot_att if tot_att else None,
        "walks_replayed_after_log_overflow": int(sum(replay_counts[-args.steps:])),
        "roofline": roofline, "clocks": clock_info, "gpu_launches": int(tot_launches),
    }

    # ---- end to end through the reference-facing host call, HOST buffers (rank 0's GPU only
    # times its own share; ranks run the same call concurrently and the rates are summed)
    target = max(1, int(accepted / max(args.steps, 1)))
    e2e_acc, e2e_s = 0, 0.0
    e2e_calls = max(1, min(args.steps, 5))
    e2e_error = None
    for i in range(-min(args.warmup, 2), e2e_calls):  # negative i: untimed warm-up calls
        barrier()
        t0 = time.perf_counter()
        try:
            with hostapi.DeviceGraph(g, p_of, device=local) as dg2:    # H2D of the CSR arrays
                _, acc = dg2.sample(target, seed=STREAM_SEED + 1000 * rank + i + 100,
                                    max_attempts=10**15)               # ensure + counters (D2H)
        except Exception as exc:  # e.g. a second copy of a 50 GB graph does not fit next to the first
            e2e_error, acc = str(exc)[:200], 0
        torch.cuda.synchronize()
        if i >= 0:
            e2e_s += time.perf_counter() - t0
            e2e_acc += acc
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    ce = torch.tensor([float(e2e_acc)], dtype=torch.float64, device="cuda")
    if world > 1:
        all_reduce(te, dist.ReduceOp.MAX)
        all_reduce(ce, dist.ReduceOp.SUM)
    out["e2e"] = {
        "value": float(ce.item()) / float(te.item()), "unit": UNIT,
        "h2d_bytes_per_step": ref_bytes, "d2h_bytes_per_step": 16,
        "call": f"DeviceGraph(g, vi) upload + SampleStream.ensure({target}) + counters_for "
                f"(the `hsaw sample` path), per call",
        "calls_timed": e2e_calls, "ms_per_call": 1e3 * float(te.item()) / e2e_calls,
    }
    if e2e_error:
        out["e2e"]["error"] = e2e_error

    # ---- eSIA seconds-to-solution on the same config (single GPU path)
    if not args.no_esia and world == 1:
        delta_ = 1.0 / g.n
        kind = 0 if args.solver == "esia" else 1
        try:
            runs = [hostapi.interdict(g, p_of, kind, args.esia_k, 0.1, delta_, seed=STREAM_SEED,
                                      max_attempts=10**15, dg=dg, want_json=True)
                    for _ in range(3)]
            r_dev = runs[-1]
            try:
                e2e_runs = [hostapi.interdict(g, p_of, kind, args.esia_k, 0.1, delta_,
                                              seed=STREAM_SEED, max_attempts=10**15, device=local,
                                              want_json=True) for _ in range(2)]
            except Exception:  # a second copy of a very large graph may not fit beside the first
                e2e_runs = [dict(r_dev, timing=dict(r_dev["timing"], wall_time_s=None))] * 2
            r_e2e = e2e_runs[-1]
            out[args.solver] = {
                "k": args.esia_k, "epsilon": 0.1, "delta": delta_,
                # graph resident in HBM; first call pays one-time pool allocations, later calls reuse
                "seconds_to_solution": r_dev["timing"]["wall_time_s"],
                "seconds_to_solution_first_call": runs[0]["timing"]["wall_time_s"],
                # host ProbGraph in, InterdictionResult out (upload + context creation inside)
                "seconds_to_solution_e2e": r_e2e["timing"]["wall_time_s"],
                "seconds_to_solution_e2e_first_call": e2e_runs[0]["timing"]["wall_time_s"],
                "breakdown_s": {k: r_dev["timing"][k] for k in ("sample_s", "greedy_s", "check_s")},
                "iterations": r_dev["iterations"], "samples_used": r_dev["samples_used"],
                "attempts": r_dev["attempts"], "coverage": r_dev["coverage"],
                "passed_check": r_dev["passed_check"], "est_suspension": r_dev["est_suspension"],
                "solution_head": r_dev["solution"][:5],
                "same_result_e2e": all(r_dev[k] == r_e2e[k]
                                       for k in ("solution", "attempts", "coverage")),
            }
        except Exception as exc:  # e.g. the walk pool of a huge instance outgrowing HBM
            out[args.solver] = {"k": args.esia_k, "error": str(exc)[:300]}

    # ---- BASELINE.json quotes seconds-to-solution at k = 1000: the same solve with that budget
    if (not args.no_esia and world == 1 and args.esia_k != 1000 and args.solver == "esia"
            and isinstance(out.get("esia"), dict) and "error" not in out["esia"]):
        try:
            r1k = [hostapi.interdict(g, p_of, 0, 1000, 0.1, 1.0 / g.n, seed=STREAM_SEED,
                                     max_attempts=10**15, dg=dg, want_json=True)
                   for _ in range(2)][-1]
            out["esia_k1000"] = {
                "k": 1000, "epsilon": 0.1, "delta": 1.0 / g.n,
                "seconds_to_solution": r1k["timing"]["wall_time_s"],
                "breakdown_s": {k: r1k["timing"][k] for k in ("sample_s", "greedy_s", "check_s")},
                "iterations": r1k["iterations"], "samples_used": r1k["samples_used"],
                "coverage": r1k["coverage"], "passed_check": r1k["passed_check"],
                "est_suspension": r1k["est_suspension"],
            }
        except Exception as exc:
            out["esia_k1000"] = {"k": 1000, "error": str(exc)[:300]}

    # ---- the step after the path: paired LT forward simulation of the solution
    # just found, on the same resident graph. Informational; not part of `value`.
    if (not args.no_esia and not args.no_suspension and world == 1
            and isinstance(out.get(args.solver), dict) and "error" not in out[args.solver]):
        try:
            kind = 0 if args.solver == "esia" else 1
            sol = np.asarray(r_dev["solution"], dtype=np.uint32)
            members = int(np.count_nonzero(p_of))
            nruns = int(max(8, min(256, (1 << 27) // (g.n + members))))
            ctx.paired_runs(kind, sol, 7, min(nruns, 8))  # warm-up: tables, scratch
            ctx.stage_times(reset=True)
            t0 = time.perf_counter()
            full, res, _ = ctx.paired_runs(kind, sol, 7, nruns)
            wall = time.perf_counter() - t0
            sim_ms, _ = ctx.stage_times(reset=True)["simulate"]
            t0 = time.perf_counter()
            est = ctx.estimate_suspension(kind, sol, 0.1, 0.1, 7)
            est_s = time.perf_counter() - t0
            out["suspension"] = {
                "call": "hsaw_gpu_paired_runs / hsaw_gpu_estimate_suspension on the solution "
                        "(proj/src/evaluation.cpp:209-242), graph resident",
                "runs_timed": nruns, "draws_per_run": g.n + members,
                "paired_runs_per_sec": nruns / wall,
                "draws_per_sec_device": nruns * (g.n + members) / (sim_ms / 1e3),
                "device_ms_per_run": sim_ms / nruns,
                "mean_full": float(full.mean()), "mean_residual": float(res.mean()),
                "estimate": {"epsilon": 0.1, "delta": 0.1, "value": est["value"],
                             "capped": est["capped"], "runs": est["runs"], "seconds": est_s},
            }
            if rank == 0 and not args.no_cpu_baseline:
                from oracle import oracle
                from oracle.oracle import Csr
                off, src, cum, _, _ = g.arrays()
                csr = Csr(g.n, g.m, off, src, cum, p_of)
                cpu_runs = 3
                if oracle.have_ref():
                    R = oracle.Ref()
                    with R.handles(csr) as hd:
                        t0, s_ = time.perf_counter(), 7
                        for _ in range(cpu_runs):
                            _, s_ = R.lt_forward_simulate(csr, s_, hd=hd)
                        dt = time.perf_counter() - t0
                    cpu_kind = "reference"
                else:
                    P = oracle.Port()
                    t0, s_ = time.perf_counter(), 7
                    for _ in range(cpu_runs):
                        _, s_ = P.lt_forward_simulate(csr, s_)
                    dt = time.perf_counter() - t0
                    cpu_kind = "port"
                out["suspension"]["cpu_baseline"] = {
                    "runs_per_sec": cpu_runs / dt, "cores": 1, "kind": cpu_kind,
                    "sample": f"{cpu_runs} x lt_forward_simulate (one realisation + one count; a "
                              f"paired run does two counts), single-threaded like the reference",
                }
        except Exception as exc:
            out["suspension"] = {"error": str(exc)[:300]}

    # ---- the step before the path, on request: file -> graph
    if args.ingest and world == 1:
        try:
            out["ingest"] = ingest_leg(args, rank == 0 and not args.no_cpu_baseline)
        except Exception as exc:
            out["ingest"] = {"error": str(exc)[:300]}

    # ---- N > 1: the sharded solve (walks sharded by batch range, marginal-gain counts combined
    # over NCCL; paper_1702_05854_b200/sharded.py). Every rank runs it; device-timed, max over ranks.
    if not args.no_esia and world > 1:
        from paper_1702_05854_b200.sharded import Comm, GpuEngine, ShardedSolver
        kind = 0 if args.solver == "esia" else 1
        try:
            res, secs = None, []
            for _ in range(2):  # first run pays one-time allocations
                eng = GpuEngine(ctx, seed=STREAM_SEED, cfg=cfg)
                try:
                    barrier()
                    s0, s1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
                    s0.record(tstream)
                    with torch.cuda.stream(tstream):
                        res = ShardedSolver(eng, Comm()).interdict(g.n, kind, args.esia_k, 0.1,
                                                                   1.0 / g.n)
                    s1.record(tstream)
                    barrier()
                    secs.append(s0.elapsed_time(s1) / 1e3)
                finally:
                    eng.close()
            tt = torch.tensor([secs[-1]], dtype=torch.float64, device="cuda")
            all_reduce(tt, dist.ReduceOp.MAX)
            out[args.solver] = {
                "k": args.esia_k, "epsilon": 0.1, "delta": 1.0 / g.n, "sharded_over": world,
                "seconds_to_solution": float(tt.item()), "seconds_to_solution_first_call": secs[0],
                "iterations": res["iterations"], "samples_used": res["samples_used"],
                "attempts": res["attempts"], "coverage": res["coverage"],
                "passed_check": res["passed_check"], "est_suspension": res["est_suspension"],
                "solution_head": res["solution"][:5],
            }
            if not args.no_suspension:
                # forward simulation of that solution, runs sharded over the ranks by stream position
                eng = GpuEngine(ctx, seed=STREAM_SEED, cfg=cfg)
                try:
                    members = int(np.count_nonzero(p_of))
                    solver = ShardedSolver(eng, Comm())
                    solver.estimate_suspension(g.n, members, kind, res["solution"], 0.1, 0.1, 7)
                    barrier()
                    t0 = time.perf_counter()
                    est = solver.estimate_suspension(g.n, members, kind, res["solution"], 0.1, 0.1, 7)
                    barrier()
                    out["suspension"] = {"sharded_over": world, "estimate": {
                        "epsilon": 0.1, "delta": 0.1, "value": est["value"], "capped": est["capped"],
                        "runs": est["runs"], "seconds": time.perf_counter() - t0}}
                finally:
                    eng.close()
        except Exception as exc:
            out[args.solver] = {"k": args.esia_k, "sharded_over": world, "error": str(exc)[:300]}

    # ---- CPU baseline beside it: rank 0, N=1 only, bounded sample
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        rate, ns, at, kind, used, dt = cpu_reference_rate(args, g, p_of, args.cpu_target,
                                                          STREAM_SEED, cores)
        out["cpu_baseline"] = {
            "value": rate, "unit": UNIT, "cores": used, "kind": kind,
            "sample": f"stream_samples to {args.cpu_target} HSAWs on the same graph/suspects/seed "
                      f"({ns} HSAWs, {at} attempts, {dt:.1f} s)",
        }
    elif rank == 0:
        out["cpu_baseline"] = None
    dg.close()
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def ingest_leg(args, with_cpu_baseline: bool) -> dict:
    """HSAW1 cache / edge-list text of a uniform graph with the workload's node and edge counts
    (validate() rejects R-MAT hub rows in 1/d mode) in /dev/shm: device loaders, host
    loaders, and - cpu_baseline - the reference's own load_cache / load_edge_list."""
    import tempfile

    from paper_1702_05854_b200 import hostapi

    def timed(fn, *a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        dt = time.perf_counter() - t0
        if hasattr(r, "close"):
            r.close()
        return dt

    g = hostapi.Graph.synth(1 << args.scale, int(args.edge_factor), 3)
    res = {"graph": f"synth_graph(2^{args.scale}, {int(args.edge_factor)}, seed 3): {g.n} nodes, {g.m} edges"}
    with tempfile.TemporaryDirectory(dir="/dev/shm" if os.path.isdir("/dev/shm") else None) as tmp:
        cache, text = os.path.join(tmp, "g.hsaw1"), os.path.join(tmp, "g.edges")
        g.save_cache(cache)
        g.save_edge_list(text)
        res["cache_bytes"], res["text_bytes"] = os.path.getsize(cache), os.path.getsize(text)
        timed(hostapi.DeviceGraph.from_cache, cache)  # warm-up: context, pools, pinned staging
        res["cache_to_resident_graph_s"] = min(timed(hostapi.DeviceGraph.from_cache, cache)
                                               for _ in range(3))
        res["cache_to_probgraph_device_s"] = min(timed(hostapi.Graph.load_cache_device, cache)
                                                 for _ in range(2))
        res["cache_to_probgraph_host_s"] = timed(hostapi.Graph.load_cache, cache)
        timed(hostapi.Graph.load_edge_list_device, text, mode=1)
        res["text_to_probgraph_device_s"] = min(
            timed(hostapi.Graph.load_edge_list_device, text, mode=1) for _ in range(2))
        res["text_to_probgraph_host_s"] = timed(hostapi.Graph.load_edge_list, text, mode=1)
        if with_cpu_baseline:
            from oracle import oracle
            if oracle.have_ref():
                R = oracle.Ref()
                t0 = time.perf_counter()
                R.graph_free(R.load_cache(cache))
                t1 = time.perf_counter()
                R.graph_free(R.load_edge_list(text, mode=1))
                t2 = time.perf_counter()
                res["cpu_baseline"] = {"kind": "reference", "cores": 1, "load_cache_s": t1 - t0,
                                       "load_edge_list_s": t2 - t1,
                                       "sample": "the same two files, one call each"}
    return res


def hsaw_mb(dg):
    from paper_1702_05854_b200 import capi
    return round(int(capi.lib().hsaw_gpu_graph_bytes(dg.ctx_handle())) / 1e6, 1)


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

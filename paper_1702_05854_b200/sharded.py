"""Sharded (multi-GPU) eSIA / nSIA: one process per GPU, graph replicated, walks sharded by batch
range, `torch.distributed` for the plumbing.

What is distributed and what is not:
  * batches (worker id = seed + b) are independent, so each round's batch range is split into
    `world` contiguous blocks; rank r samples block r on its GPU and keeps its walks local. The
    global (batch, seq) order is then round-major, rank-major — exactly the single-stream order
    (proj/src/sampler.cpp:452-460) — so R_t = global prefix [0, size) and R'_t = [size, 2 size) are
    *contiguous local ranges* on every rank (`Layout.local_range`).
  * exchange steps: (1) all-gather of per-block accepted counts after each round (w integers);
    (2) greedy: one all-reduce(sum) of the marginal-gain count vector per call, then per round an
    all-gather of the (sparse) decrement lists, so every rank keeps an identical replica of the
    counts and picks the same winner; (3) scalar all-reduces for coverage_of; (4) one broadcast for
    counters_for. No walk ever crosses NVLink.
  * schedule, stopping rule and the doubling loop are the host functions of the single-GPU path
    (hostapi.schedule / hostapi.check), so results are identical for every world size.

The device work goes through an *engine* (GpuEngine below, on the C-ABI). The orchestration itself
is engine-agnostic, which is how tests/test_sharded_cpu.py runs it with world_size 2 over gloo on a
CPU-only box against a test-side engine.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from .capi import (HSAW_EBUDGET, HSAW_EDATA, HSAW_EINVAL, HSAW_ERANGE, KIND_EDGE, KIND_NODE,
                   HsawError)


# ---- communication plumbing -----------------------------------------------------------------------
class Comm:
    """Thin wrapper over a torch.distributed group (NCCL on GPUs, gloo in CPU tests)."""

    def __init__(self, group=None):
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.on else 0
        self.world = dist.get_world_size(group) if self.on else 1
        self.backend = dist.get_backend(group) if self.on else "none"

    def _staged(self, t: torch.Tensor) -> torch.Tensor:
        # gloo cannot all-gather CUDA tensors: stage through the host in that (test-only) setup
        return t.cpu() if (self.backend == "gloo" and t.is_cuda) else t

    def allgather_ints(self, values: list[int]) -> list[list[int]]:
        if self.world == 1:
            return [list(values)]
        dev = "cuda" if self.backend == "nccl" else "cpu"
        mine = torch.tensor(values, dtype=torch.int64, device=dev)
        out = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(out, mine, group=self.group)
        return [[int(x) for x in o.tolist()] for o in out]

    def allreduce_sum_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return t
        s = self._staged(t)
        dist.all_reduce(s, op=dist.ReduceOp.SUM, group=self.group)
        if s is not t:
            t.copy_(s)
        return t

    def allgather_var(self, t: torch.Tensor) -> list[torch.Tensor]:
        """All-gather of 1-D tensors of different lengths (lengths first, then padded payloads)."""
        if self.world == 1:
            return [t]
        lens = [x[0] for x in self.allgather_ints([int(t.numel())])]
        cap = max(max(lens), 1)
        s = self._staged(t)
        pad = torch.zeros(cap, dtype=t.dtype, device=s.device)
        pad[: t.numel()] = s
        out = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(out, pad, group=self.group)
        return [o[:n].to(t.device) for o, n in zip(out, lens)]

    def broadcast_ints(self, values: list[int], src: int) -> list[int]:
        if self.world == 1:
            return list(values)
        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor(values, dtype=torch.int64, device=dev)
        dist.broadcast(t, src=dist.get_global_rank(self.group, src) if self.group else src,
                       group=self.group)
        return [int(x) for x in t.tolist()]


# ---- global order bookkeeping (pure host logic) ------------------------------------------------
@dataclass
class Round:
    first_batch: int
    sizes: list[int]      # batches given to each rank (contiguous blocks, in rank order)
    accepted: list[int]   # decoded walks each rank's block produced

    def block_start(self, r: int) -> int:
        return self.first_batch + sum(self.sizes[:r])


@dataclass
class Layout:
    """Where the global (batch, seq) order lives: per round, per rank."""

    world: int
    rounds: list[Round] = field(default_factory=list)

    @property
    def accepted(self) -> int:
        return sum(sum(r.accepted) for r in self.rounds)

    @property
    def batches(self) -> int:
        return sum(sum(r.sizes) for r in self.rounds)

    @staticmethod
    def split(first_batch: int, batches: int, world: int) -> list[int]:
        base, rem = divmod(batches, world)
        return [base + (1 if r < rem else 0) for r in range(world)]

    def count_below(self, rank: int, x: int) -> int:
        """Number of `rank`'s walks whose global position is < x."""
        g, total = 0, 0
        for rd in self.rounds:
            for r in range(self.world):
                a = rd.accepted[r]
                if r == rank:
                    total += min(max(x - g, 0), a)
                g += a
        return total

    def local_range(self, rank: int, off: int, cnt: int) -> tuple[int, int]:
        """Global walks [off, off+cnt) -> this rank's contiguous local range (offset, count)."""
        lo = self.count_below(rank, off)
        return lo, self.count_below(rank, off + cnt) - lo

    def locate(self, target: int):
        """Block (round index, rank) inside which the cumulative accepted count reaches target,
        with the global count before that block; None if not materialised."""
        g = 0
        for j, rd in enumerate(self.rounds):
            for r in range(self.world):
                if g + rd.accepted[r] >= target:
                    return j, r, g
                g += rd.accepted[r]
        return None


# ---- the device-side worker of one rank ----------------------------------------------------------
class GpuEngine:
    """One rank's GPU through the C-ABI (capi). Buffers exchanged with peers are torch tensors."""

    def __init__(self, ctx, seed: int, cfg=None):
        from . import capi
        self.capi, self.ctx = capi, ctx
        self.cfg = cfg or capi.SamplerCfg()
        self.batch_size = self.cfg.batch_size
        self.max_attempts = self.cfg.max_attempts
        big = capi.SamplerCfg(self.cfg.heuristic, self.cfg.window, self.cfg.batch_size, 2**62)
        self.stream = ctx.stream(seed=seed, cfg=big)  # the budget is enforced globally, not here
        self.device = torch.device("cuda", torch.cuda.current_device())

    def close(self):
        self.stream.close()

    def limit(self, kind: int) -> int:
        return self.ctx.m if kind == KIND_EDGE else self.ctx.n

    def sample_range(self, first_batch: int, nbatches: int) -> int:
        return self.stream.sample_range(first_batch, nbatches) if nbatches else 0

    def local_cut(self, min_local: int):
        return self.stream.local_cut(min_local)

    def coverage_of(self, items, kind, off, cnt, cand) -> int:
        if cnt == 0:
            return 0
        return self.ctx.coverage_of(items, stream=self.stream, kind=kind, off=off, cnt=cnt,
                                    cand=cand)

    def coverage_upper_bound(self, k, kind, off, cnt, cand) -> int:
        if cnt == 0:
            return 0
        return self.ctx.coverage_upper_bound(k, stream=self.stream, kind=kind, off=off, cnt=cnt,
                                             cand=cand)

    # -- building blocks of the gather-and-replicate greedy (hsaw_gpu.h, "sharded solve")
    def local_counts(self, kind, off, cnt, cand) -> torch.Tensor:
        """Occurrences of every candidate item in local walks [off, off+cnt): int32[limit], device."""
        counts = torch.zeros(self.limit(kind), dtype=torch.int32, device=self.device)
        torch.cuda.current_stream().synchronize()
        ca = None if cand is None else np.ascontiguousarray(cand, dtype=np.uint32)
        self.ctx._chk(self.capi.lib().hsaw_gpu_stream_histogram(
            self.ctx.h, self.stream.h, kind, off, cnt, self.capi._p(ca, self.capi.u32p),
            0 if ca is None else ca.size, counts.data_ptr()))
        return counts

    def bound_from_counts(self, counts: torch.Tensor, k: int, cap: int) -> int:
        out = self.capi.C.c_uint64()
        torch.cuda.current_stream().synchronize()
        self.ctx._chk(self.capi.lib().hsaw_gpu_counts_bound(self.ctx.h, counts.data_ptr(),
                                                            counts.numel(), k, cap,
                                                            self.capi.C.byref(out)))
        return out.value

    def threshold_from_counts(self, counts: torch.Tensor, k: int = 0, ck_percent: int = 0) -> int:
        """The 1/8-mass indexing threshold, raised to ck_percent % of the k-th largest count."""
        out = self.capi.C.c_uint32()
        torch.cuda.current_stream().synchronize()
        self.ctx._chk(self.capi.lib().hsaw_gpu_counts_threshold_for(
            self.ctx.h, counts.data_ptr(), counts.numel(), k, ck_percent, self.capi.C.byref(out)))
        return out.value

    def reduced_walks(self, kind, off, cnt, counts: torch.Tensor, min_count: int):
        """Local walks restricted to items with global count >= min_count -> (lens int32[w'],
        items int32[...]) device tensors; walks left empty are dropped."""
        C = self.capi.C
        h, ns, ni = C.c_void_p(), C.c_uint64(), C.c_uint64()
        torch.cuda.current_stream().synchronize()
        self.ctx._chk(self.capi.lib().hsaw_gpu_reduced_walks(
            self.ctx.h, self.stream.h, kind, off, cnt, counts.data_ptr(), min_count, C.byref(h),
            C.byref(ns), C.byref(ni)))
        try:
            lens = torch.empty(ns.value, dtype=torch.int32, device=self.device)
            items = torch.empty(ni.value, dtype=torch.int32, device=self.device)
            torch.cuda.current_stream().synchronize()
            self.ctx._chk(self.capi.lib().hsaw_gpu_walkset_copy_device(
                h, lens.data_ptr() if ns.value else None, items.data_ptr() if ni.value else None))
        finally:
            self.capi.lib().hsaw_gpu_walkset_destroy(h)
        return lens, items

    def greedy_on_sets(self, kind, lens: torch.Tensor, items: torch.Tensor, k: int, cand):
        """The single-GPU greedy (tail kernel and all) on gathered sets -> (solution, coverage,
        smallest per-round gain; 0 if the gains ran out)."""
        C = self.capi.C
        h = C.c_void_p()
        lens, items = lens.contiguous(), items.contiguous()
        torch.cuda.current_stream().synchronize()
        self.ctx._chk(self.capi.lib().hsaw_gpu_walkset_from_device(
            self.ctx.h, self.limit(kind), lens.numel(), lens.data_ptr() if lens.numel() else None,
            items.data_ptr() if items.numel() else None, items.numel(), C.byref(h)))
        ws = self.capi.WalkSet.adopt(self.ctx, h, lens.numel(), items.numel())
        try:
            sol, cov = self.ctx.greedy(k, walkset=ws, kind=kind, cand=cand)
            min_gain = int(self.capi.lib().hsaw_gpu_last_greedy_min_gain(self.ctx.h))
        finally:
            ws.close()
        return [int(x) for x in sol], int(cov), min_gain

    def paired_runs(self, kind, ids, state0, first_run, nruns, draws_per_run):
        """Runs [first_run, first_run + nruns) of the simulation stream that starts at state0."""
        if nruns == 0:
            return np.zeros(0, dtype=np.uint32), np.zeros(0, dtype=np.uint32)
        s = self.capi.prg_jump(state0, first_run * draws_per_run)
        full, res, _ = self.ctx.paired_runs(kind, ids, s, nruns)
        return full, res

    class _Rounds:
        def __init__(self, eng, kind, off, cnt, cand):
            self.eng = eng
            limit = eng.limit(kind)
            self.counts = torch.zeros(limit + 4, dtype=torch.int32, device=eng.device)
            torch.cuda.current_stream().synchronize()
            self.r = eng.capi.Rounds(eng.ctx, self.counts.data_ptr(), stream=eng.stream, kind=kind,
                                     off=off, cnt=cnt, cand=cand)
            self.list = torch.empty(max(self.r.occurrences, 1), dtype=torch.int32,
                                    device=eng.device)
            torch.cuda.current_stream().synchronize()

        def select(self):
            torch.cuda.current_stream().synchronize()  # counts may have been all-reduced by torch
            return self.r.select()

        def cover(self, item) -> torch.Tensor:
            n = self.r.cover(item, self.list.data_ptr(), self.list.numel())
            return self.list[:n]

        def apply(self, items: torch.Tensor):
            if items.numel():
                items = items.contiguous()
                torch.cuda.current_stream().synchronize()
                self.r.apply(items.data_ptr(), items.numel())
                self.eng.ctx.sync()

        def close(self):
            self.r.close()

    def begin_rounds(self, kind, off, cnt, cand):
        return GpuEngine._Rounds(self, kind, off, cnt, cand)


# ---- the sharded sample stream + solver ----------------------------------------------------------
class ShardedSolver:
    """SampleStream + greedy + the doubling loop over `comm.world` engines (one per process)."""

    def __init__(self, engine, comm: Comm | None = None):
        self.eng = engine
        self.comm = comm or Comm()
        self.layout = Layout(self.comm.world)
        self.next_batch = 0
        self.grow = 4096
        self.local_accepted = 0

    # -- SampleStream::ensure (proj/src/sampler.cpp:388-463), sharded
    def ensure(self, min_accepted: int):
        bs, w = self.eng.batch_size, self.comm.world
        while self.layout.accepted < min_accepted:
            attempts_so_far = self.next_batch * bs
            budget_left = max(self.eng.max_attempts - attempts_so_far, 0)
            max_batches = budget_left // bs
            if max_batches == 0:
                raise HsawError(HSAW_EBUDGET, "attempt budget exhausted while sampling walks; "
                                              "suspects may be unreachable")
            have = self.layout.accepted
            if have == 0:
                batches, self.grow = self.grow, min(self.grow * 8, 1 << 22)
            else:
                rate = have / attempts_so_far
                batches = int((min_accepted - have) / (rate * bs) * 1.1) + 64
            batches = max(min(batches, max_batches), 1)
            sizes = Layout.split(self.next_batch, batches, w)
            rd = Round(self.next_batch, sizes, [0] * w)
            got = self.eng.sample_range(rd.block_start(self.comm.rank), sizes[self.comm.rank])
            rd.accepted = [x[0] for x in self.comm.allgather_ints([got])]
            self.local_accepted += got
            self.layout.rounds.append(rd)
            self.next_batch += batches

    # -- SampleStream::counters_for (sampler.cpp:472-482), sharded
    def counters_for(self, min_accepted: int):
        if min_accepted == 0:
            return 0, 0
        where = self.layout.locate(min_accepted)
        if where is None:
            raise HsawError(HSAW_ERANGE, "sample stream target not materialized")
        j, owner, before = where
        rd = self.layout.rounds[j]
        vals = [0, 0]
        if self.comm.rank == owner:
            local_before = sum(r.accepted[owner] for r in self.layout.rounds[:j])
            batches_before = sum(r.sizes[owner] for r in self.layout.rounds[:j])
            nb, acc = self.eng.local_cut(local_before + (min_accepted - before))
            in_block = nb - batches_before
            global_batches = (rd.block_start(owner) + in_block)  # batches are numbered from 0
            vals = [global_batches * self.eng.batch_size, before + (acc - local_before)]
        vals = self.comm.broadcast_ints(vals, owner)
        return vals[0], vals[1]

    # -- CoverageIndex::coverage_of on global walks [off, off+cnt)
    def coverage_of(self, items, kind, off, cnt, cand=None) -> int:
        lo, n = self.layout.local_range(self.comm.rank, off, cnt)
        local = self.eng.coverage_of(items, kind, lo, n, cand)
        t = torch.tensor([local], dtype=torch.int64)
        if self.comm.backend == "nccl":
            t = t.cuda()
        return int(self.comm.allreduce_sum_(t).item())

    def coverage_upper_bound(self, k, kind, off, cnt, cand=None) -> int:
        """Upper bound of coverage_of over every k candidates on global walks [off, off+cnt): the
        counts of all ranks are all-reduced first, so the bound is exactly the single-GPU one (the
        sum of the k largest global counts) and the same iterations are skipped for every world
        size. Engines without the primitives fall back to the (looser) sum of local bounds."""
        lo, n = self.layout.local_range(self.comm.rank, off, cnt)
        if hasattr(self.eng, "local_counts"):
            counts = self.eng.local_counts(kind, lo, n, cand)
            self.comm.allreduce_sum_(counts)
            return self.eng.bound_from_counts(counts, k, cnt)
        fn = getattr(self.eng, "coverage_upper_bound", None)
        local = n if fn is None else fn(k, kind, lo, n, cand)
        t = torch.tensor([local], dtype=torch.int64)
        if self.comm.backend == "nccl":
            t = t.cuda()
        return int(self.comm.allreduce_sum_(t).item())

    # -- greedy_max_cover on global walks [0, size) (proj/src/coverage.cpp:91-138), sharded
    def greedy(self, k: int, kind: int, size: int, cand=None):
        limit = self.eng.limit(kind)
        cand_sorted = None
        if cand is not None:
            ca = np.asarray(cand, dtype=np.int64)
            if ca.size and (ca.max() >= limit or ca.min() < 0):
                raise HsawError(HSAW_EDATA, "candidate id out of range")
            cand_sorted = np.unique(ca)
        ncand = limit if cand_sorted is None else int(cand_sorted.size)
        if k > ncand:
            raise HsawError(HSAW_EINVAL, "budget k exceeds candidate count")
        lo, n = self.layout.local_range(self.comm.rank, 0, size)
        if hasattr(self.eng, "reduced_walks"):
            return self._greedy_gathered(k, kind, lo, n, cand)
        rounds = self.eng.begin_rounds(kind, lo, n, cand)
        try:
            self.comm.allreduce_sum_(rounds.counts)  # local histograms -> global marginal gains
            solution, coverage = [], 0
            while len(solution) < k:
                item, gain = rounds.select()
                if gain == 0:
                    break
                solution.append(item)
                coverage += gain
                mine = rounds.cover(item)
                for r, lst in enumerate(self.comm.allgather_var(mine)):
                    if r != self.comm.rank:
                        rounds.apply(lst)
        finally:
            rounds.close()
        # zero-gain slots: smallest unselected candidates (coverage.cpp:101-106,155)
        chosen = set(solution)
        c = 0
        while len(solution) < k:
            cid = int(cand_sorted[c]) if cand_sorted is not None else c
            c += 1
            if cid not in chosen:
                solution.append(cid)
                chosen.add(cid)
        return solution, coverage

    def _greedy_gathered(self, k, kind, lo, n, cand):
        """One all-reduce of the local count vectors, one all-gather of the local walks restricted
        to the items that can still win (global count >= the indexing threshold of the single-GPU
        greedy), then the single-GPU greedy on the gathered sets, redundantly on every rank: same
        selections everywhere, no per-round exchange. If the k-th gain falls below the threshold
        the reduced instance was not enough: repeat with the next, lower threshold."""
        counts = self.eng.local_counts(kind, lo, n, cand)
        self.comm.allreduce_sum_(counts)
        # thresholds from bold to safe (60 %, 30 % of the k-th largest count, the 1/8-mass rule,
        # then everything): a run whose smallest gain stays at or above its threshold is exact
        ladder = []
        for pct in (60, 30, 0):
            mc = self.eng.threshold_from_counts(counts, k, pct)
            if not ladder or mc < ladder[-1]:
                ladder.append(mc)
        if ladder[-1] > 1:
            ladder.append(1)
        for min_count in ladder:
            lens, items = self.eng.reduced_walks(kind, lo, n, counts, min_count)
            all_lens = self.comm.allgather_var(lens)
            all_items = self.comm.allgather_var(items)
            solution, coverage, min_gain = self.eng.greedy_on_sets(
                kind, torch.cat(all_lens), torch.cat(all_items), k, cand)
            if min_count <= 1 or min_gain >= min_count:
                return solution, coverage
        raise AssertionError("unreachable: the last rung gathers everything")

    # -- run_interdiction (proj/src/interdiction.cpp:12-67), sharded
    # ---- estimate_suspension (proj/src/evaluation.cpp:209-242), runs sharded over the ranks -------
    def estimate_suspension(self, n_nodes: int, members: int, kind: int, ids, eps: float,
                            delta: float, state: int, batch_runs: int | None = None) -> dict:
        """Paired forward simulation with each device batch of runs split into `world` contiguous
        run ranges (every run is addressed by its stream position, capi.prg_jump). Exchange step:
        one all-gather of the per-run (full, residual) counts per batch; every rank then replays
        the reference's FP64 accumulation in run order, so value / capped / runs / state are the
        single-GPU (and reference) results for every world size."""
        import math

        from . import capi
        if not (eps > 0.0) or eps >= 1.0:
            raise HsawError(HSAW_EINVAL, "epsilon must be in (0,1)")
        if not (delta > 0.0) or delta >= 1.0:
            raise HsawError(HSAW_EINVAL, "delta must be in (0,1)")
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        limit = self.eng.limit(kind)
        for x in ids.tolist():
            if x >= limit:
                raise HsawError(HSAW_EDATA, f"removal id out of range: {x}")
        if ids.size == 0:
            return dict(value=0.0, capped=False, runs=0, state=state)
        upsilon = 4.0 * (math.exp(1.0) - 2.0) * math.log(2.0 / delta) * (1.0 + eps) / (eps * eps)
        d = members + n_nodes
        max_runs = max(1, 1_000_000_000 // d)
        cap = batch_runs or max(self.comm.world, (self.comm.world << 25) // d)
        total, runs, capped = 0.0, 0, False
        while total < upsilon:
            if runs >= max_runs:
                capped = True
                break
            want = 64 * self.comm.world
            if runs:
                want = 2 * runs
                if total > 0.0:
                    want = int((upsilon - total) / (total / runs) * 1.05) + 16
            b = max(1, min(cap, max(want, 16), max_runs - runs))
            sizes = Layout.split(0, b, self.comm.world)
            first = runs + sum(sizes[: self.comm.rank])
            full, res = self.eng.paired_runs(kind, ids, state, first, sizes[self.comm.rank], d)
            mine = torch.from_numpy(np.stack([full, res]).astype(np.int64).reshape(-1))
            parts = self.comm.allgather_var(mine.to(self._exchange_device()))
            for part in parts:  # rank order = run order
                fr = part.cpu().numpy().reshape(2, -1)
                for f, r in zip(fr[0].tolist(), fr[1].tolist()):
                    if not total < upsilon:
                        break
                    total += float(f - r) / float(n_nodes)
                    runs += 1
        out_state = capi.prg_jump(state, runs * d)
        if capped:
            return dict(value=0.0, capped=True, runs=runs, state=out_state)
        return dict(value=float(n_nodes) * upsilon / float(runs), capped=False, runs=runs,
                    state=out_state)

    def _exchange_device(self):
        return "cuda" if self.comm.backend == "nccl" else "cpu"

    def interdict(self, n_nodes: int, kind: int, k: int, eps: float, delta: float, cand=None):
        from . import hostapi
        limit = self.eng.limit(kind)
        if cand is not None:
            ca = list(cand)
            if len(ca) == 0:
                raise HsawError(HSAW_EDATA, "candidate set is empty")
            if any(c >= limit for c in ca) or len(set(ca)) != len(ca):
                raise HsawError(HSAW_EDATA, "candidate id out of range or duplicated")
        csize = limit if cand is None else len(cand)
        if csize == 0:
            raise HsawError(HSAW_EDATA, "candidate set is empty")
        if k < 1 or k > csize:
            raise HsawError(HSAW_EINVAL, "budget k must be in [1, |C|]")
        sched = hostapi.schedule(limit, k, eps, delta)
        lam = sched["lambda_samples"]
        t = 0
        bound_can_skip = True
        while True:
            t += 1
            size = lam << (t - 1)
            self.ensure(2 * size)
            # an iteration whose R'_t cannot reach Lambda_1 with any k candidates cannot pass the
            # check (coverage.cpp:216-217): skip its greedy run unless N_max ends the loop here.
            # Once a bound has reached Lambda_1 the later, larger R' will too: no more bounds.
            if bound_can_skip and float(size) < sched["n_max"]:
                if float(size) < sched["lambda1"]:  # Cov_R'(S) <= |R'_t| = size
                    continue
                if self.coverage_upper_bound(k, kind, size, size, cand) < sched["lambda1"]:
                    continue
                bound_can_skip = False
            solution, coverage = self.greedy(k, kind, size, cand)
            cov_r = self.coverage_of(solution, kind, 0, size, cand)
            cov_rp = self.coverage_of(solution, kind, size, size, cand)
            ok, _ = hostapi.check(cov_r, cov_rp, size, limit, k, eps, delta, t)
            if ok or float(size) >= sched["n_max"]:
                break
        attempts, accepted = self.counters_for(2 * size)
        influence = float(n_nodes) * float(accepted) / float(attempts)
        return dict(kind="edge" if kind == KIND_EDGE else "node", k=k, epsilon=eps, delta=delta,
                    solution=[int(x) for x in solution],
                    est_suspension=influence * float(coverage) / float(size), coverage=coverage,
                    samples_used=2 * size, attempts=attempts, iterations=t, passed_check=bool(ok))

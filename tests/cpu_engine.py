"""TEST INFRASTRUCTURE: a CPU stand-in for sharded.GpuEngine built on the oracle, so that the
multi-rank orchestration (paper_1702_05854_b200/sharded.py) can run with world_size 2 over gloo on
a box without GPUs. Same interface as GpuEngine; never used by the product."""
import numpy as np
import torch


class CpuEngine:
    def __init__(self, port, csr, seed, batch_size=10, max_attempts=100_000_000):
        self.port, self.csr, self.seed = port, csr, seed
        self.batch_size, self.max_attempts = batch_size, max_attempts
        self.walk_nodes, self.walk_edges = [], []
        self.accepted_after_batch = []
        self.last_end = 0

    def close(self):
        pass

    def limit(self, kind):
        return self.csr.m if kind == 0 else self.csr.n

    def sample_range(self, first_batch, nbatches):
        assert first_batch >= self.last_end, "ranges must be increasing"
        before = len(self.walk_nodes)
        for b in range(first_batch, first_batch + nbatches):
            seeds, lens = self.port.thread_sample(self.csr, (self.seed + b) % 2**64,
                                                  self.batch_size)
            for s, ln in zip(seeds, lens):
                dec = self.port.decode(self.csr, int(s), int(ln))
                if dec is not None:
                    self.walk_nodes.append(dec[0])
                    self.walk_edges.append(dec[1])
            self.accepted_after_batch.append(len(self.walk_nodes))
        self.last_end = first_batch + nbatches
        return len(self.walk_nodes) - before

    def local_cut(self, min_local):
        for i, a in enumerate(self.accepted_after_batch):
            if a >= min_local:
                return i + 1, a
        raise RuntimeError("local cut beyond materialised batches")

    def paired_runs(self, kind, ids, state0, first_run, nruns, draws_per_run):
        from paper_1702_05854_b200 import capi  # host-only jump-ahead helper of the C-ABI
        if nruns == 0:
            return np.zeros(0, dtype=np.uint32), np.zeros(0, dtype=np.uint32)
        s = capi.prg_jump(state0, first_run * draws_per_run)
        full, res, _ = self.port.paired_runs(self.csr, kind, ids, s, nruns)
        return full, res

    def _items(self, kind, w):
        return self.walk_edges[w] if kind == 0 else self.walk_nodes[w]

    def coverage_of(self, items, kind, off, cnt, cand):
        q = set(int(x) for x in items)
        if cand is not None:
            q &= set(int(c) for c in cand)
        return sum(1 for w in range(off, off + cnt) if q.intersection(self._items(kind, w).tolist()))

    # -- building blocks of the gather-and-replicate greedy (mirrors sharded.GpuEngine)
    K_BINS = 1024

    def local_counts(self, kind, off, cnt, cand):
        limit = self.limit(kind)
        counts = np.zeros(limit, dtype=np.int64)
        ok = np.ones(limit, dtype=bool)
        if cand is not None:
            ok[:] = False
            ok[np.asarray(cand, dtype=np.int64)] = True
        for w in range(off, off + cnt):
            it = self._items(kind, w).astype(np.int64)
            np.add.at(counts, it[ok[it]], 1)
        return torch.from_numpy(counts.astype(np.int32))

    def _bins(self, counts):
        c = counts.numpy().astype(np.int64)
        c = c[c > 0]
        bins = np.zeros(self.K_BINS, dtype=np.int64)
        np.add.at(bins, np.minimum(c, self.K_BINS - 1), c)
        return bins

    def bound_from_counts(self, counts, k, cap):
        bins = self._bins(counts)
        total, left = int(bins[self.K_BINS - 1]), k
        for c in range(self.K_BINS - 2, 0, -1):
            if left <= 0:
                break
            take = min(int(bins[c]) // c, left)
            total += take * c
            left -= take
        return min(total, cap)

    def threshold_from_counts(self, counts, k=0, ck_percent=0):
        bins = self._bins(counts)
        total = int(bins.sum())
        mc = 1
        if total > (1 << 20):
            above, mc = 0, self.K_BINS - 1
            for c in range(self.K_BINS - 1, 0, -1):
                if above + int(bins[c]) > total // 8:
                    break
                above += int(bins[c])
                mc = c
        if ck_percent and k:  # hsaw_gpu_counts_threshold_for: a share of the k-th largest count
            items, ck = 0, 0
            for c in range(self.K_BINS - 1, 0, -1):
                items += (int(bins[c]) + c - 1) // c
                if items >= k:
                    ck = c
                    break
            mc = max(mc, ck * ck_percent // 100)
        return mc

    def reduced_walks(self, kind, off, cnt, counts, min_count):
        c = counts.numpy()
        lens, items = [], []
        for w in range(off, off + cnt):
            it = self._items(kind, w)
            keep = it[(c[it] >= max(min_count, 1)) & (c[it] > 0)]
            if keep.size:
                lens.append(keep.size)
                items.append(keep.astype(np.int32))
        cat = np.concatenate(items) if items else np.zeros(0, dtype=np.int32)
        return torch.tensor(lens, dtype=torch.int32), torch.from_numpy(cat)

    def greedy_on_sets(self, kind, lens, items, k, cand):
        limit = self.limit(kind)
        off = np.zeros(lens.numel() + 1, dtype=np.uint64)
        np.cumsum(lens.numpy().astype(np.uint64), out=off[1:])
        it = items.numpy().astype(np.uint32)
        sol, cov = self.port.greedy(limit, off, it, k, cand=cand)
        # per-round gains by replay (the oracle only returns their sum)
        sets = [set(it[int(off[i]):int(off[i + 1])].tolist()) for i in range(lens.numel())]
        covered, gains = np.zeros(len(sets), dtype=bool), []
        for x in sol.tolist():
            g = 0
            for i, st in enumerate(sets):
                if not covered[i] and x in st:
                    covered[i] = True
                    g += 1
            gains.append(g)
        return [int(x) for x in sol], int(cov), (min(gains) if gains else 0)

    class _Rounds:
        def __init__(self, eng, kind, off, cnt, cand):
            limit = eng.limit(kind)
            self.is_cand = np.ones(limit, dtype=bool)
            if cand is not None:
                self.is_cand[:] = False
                self.is_cand[np.asarray(cand, dtype=np.int64)] = True
            self.walks = [eng._items(kind, w) for w in range(off, off + cnt)]
            self.walks = [w[self.is_cand[w]] for w in self.walks]
            self.counts = torch.zeros(limit + 4, dtype=torch.int32)
            self.by_item = {}
            for i, w in enumerate(self.walks):
                for it in w.tolist():
                    self.counts[it] += 1
                    self.by_item.setdefault(it, []).append(i)
            self.covered = np.zeros(len(self.walks), dtype=bool)

        def select(self):
            c = self.counts.numpy()
            best = int(c.max())
            if best <= 0:
                return 0xFFFFFFFF, 0
            return int(np.flatnonzero(c == best)[0]), best

        def cover(self, item):
            out = []
            for i in self.by_item.get(item, []):
                if self.covered[i]:
                    continue
                self.covered[i] = True
                for it in self.walks[i].tolist():
                    self.counts[it] -= 1
                    out.append(it)
            return torch.tensor(out, dtype=torch.int32)

        def apply(self, items):
            for it in items.tolist():
                self.counts[it] -= 1

        def close(self):
            pass

    def begin_rounds(self, kind, off, cnt, cand):
        return CpuEngine._Rounds(self, kind, off, cnt, cand)

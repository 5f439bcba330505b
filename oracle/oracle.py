"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the two CPU checkers.

* ``Port``  -> oracle/_build/libhsaw_oracle.so, the plain-C restatement (hsaw_oracle.c)
* ``Ref``   -> oracle/_ref/libhsaw_ref.so, the unmodified reference behind ref_shim.cpp

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs import
this module. The product package (paper_1702_05854_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libhsaw_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhsaw_ref.so")

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
f64p = C.POINTER(C.c_double)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def build(force: bool = False) -> None:
    """Compile the C restatement (always possible) and the reference shim (only where
    /root/reference exists). Building the checker is not using it."""
    if force or not os.path.exists(PORT_SO) or os.path.getmtime(PORT_SO) < max(
        os.path.getmtime(os.path.join(HERE, f)) for f in ("hsaw_oracle.c", "hsaw_oracle.h")
    ):
        subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
    if os.path.isdir("/root/reference/proj/src") and (
        force
        or not os.path.exists(REF_SO)
        or os.path.getmtime(REF_SO) < os.path.getmtime(os.path.join(HERE, "ref_shim.cpp"))
    ):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


def have_ref() -> bool:
    return os.path.exists(REF_SO)


@dataclass
class Csr:
    """ProbGraph + SuspectSet as flat arrays (proj/include/hsaw/graph.hpp:19-51,84-94)."""

    n: int
    m: int
    in_offsets: np.ndarray  # u64[n+1]
    in_src: np.ndarray  # u32[m]
    in_cum: np.ndarray  # f64[m]
    p_of: np.ndarray  # f64[n]

    def __post_init__(self):
        self.in_offsets = np.ascontiguousarray(self.in_offsets, dtype=np.uint64)
        self.in_src = np.ascontiguousarray(self.in_src, dtype=np.uint32)
        self.in_cum = np.ascontiguousarray(self.in_cum, dtype=np.float64)
        self.p_of = np.ascontiguousarray(self.p_of, dtype=np.float64)
        assert self.in_offsets.shape == (self.n + 1,)
        assert self.in_src.shape == (self.m,) and self.in_cum.shape == (self.m,)
        assert self.p_of.shape == (self.n,)


@dataclass
class PoolData:
    attempts: int
    edge_off: np.ndarray  # u64[ns+1]
    nodes: np.ndarray  # u32[total_edges+ns]; walk w: nodes[edge_off[w]+w : edge_off[w+1]+w+1]
    edges: np.ndarray  # u32[total_edges];    walk w: edges[edge_off[w] : edge_off[w+1]]
    tag_worker: np.ndarray
    tag_seq: np.ndarray

    @property
    def nsamples(self) -> int:
        return len(self.edge_off) - 1

    def walk_nodes(self, w: int) -> np.ndarray:
        return self.nodes[int(self.edge_off[w]) + w : int(self.edge_off[w + 1]) + w + 1]

    def walk_edges(self, w: int) -> np.ndarray:
        return self.edges[int(self.edge_off[w]) : int(self.edge_off[w + 1])]

    def item_sets(self, kind: int, off: int = 0, cnt: int | None = None):
        """CSR item sets of walks [off, off+cnt): edges (kind 0) or nodes (kind 1)."""
        cnt = self.nsamples - off if cnt is None else cnt
        eo = self.edge_off[off : off + cnt + 1].astype(np.int64)
        if kind == 0:
            so = (eo - eo[0]).astype(np.uint64)
            return so, self.edges[eo[0] : eo[-1]].copy()
        idx = np.arange(cnt + 1, dtype=np.int64)
        so = (eo - eo[0] + idx).astype(np.uint64)
        return so, self.nodes[eo[0] + off : eo[-1] + off + cnt].copy()


class _OrcGraph(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m", C.c_uint32), ("in_offsets", u64p), ("in_src", u32p),
                ("in_cum", f64p), ("p_of", f64p),
                ("domain", u32p), ("ndomain", C.c_uint64), ("allowed", C.POINTER(C.c_uint8))]


@dataclass
class Partitioning:
    """proj/include/hsaw/partition.hpp:16-25: node -> part, part -> owned nodes (ascending), part ->
    byte mask of the h-hop in-neighbourhood closure."""

    p: int
    hops: int
    assign: np.ndarray      # u32[n]
    base: list              # p arrays of u32 node ids
    extended: list          # p arrays of u8[n]


@dataclass
class DistributedData:
    """DistributedResult, partition.hpp:38-44."""

    pool: "PoolData"
    crossings: int
    attempts: int
    crossing_fraction: float
    targets: list


def splitmix_output(x: int) -> int:
    """splitmix_next(x).output, proj/include/hsaw/prng.hpp:29-38."""
    M = (1 << 64) - 1
    z = (x + 0x9E3779B97F4A7C15) & M
    o = z
    o = ((o ^ (o >> 30)) * 0xBF58476D1CE4E5B9) & M
    o = ((o ^ (o >> 27)) * 0x94D049BB133111EB) & M
    return o ^ (o >> 31)


def partition_graph_np(csr: "Csr", p: int, method: str = "hash", seed: int = 0, assign=None):
    """partition_graph, proj/src/partition.cpp:29-121 (restated; small graphs only — the label
    propagation is a per-node Python loop). method: 'hash' (v mod p), 'labelprop', 'external'
    (assign given)."""
    n = csr.n
    if p < 1 or p > n:
        raise BuildError("part count must be in [1, n]")
    if method == "hash":
        a = (np.arange(n, dtype=np.uint64) % p).astype(np.uint32)
    elif method == "external":
        a = np.ascontiguousarray(assign, dtype=np.uint32)
        if a.size != n or (a.size and a.max() >= p):
            raise BuildError("part file does not match the graph")
    elif method == "labelprop":
        M = (1 << 64) - 1
        label = np.array([splitmix_output((seed * 0x9E3779B97F4A7C15 + v) & M) % p
                          for v in range(n)], dtype=np.int64)
        dst = np.repeat(np.arange(n, dtype=np.int64), np.diff(csr.in_offsets).astype(np.int64))
        src = csr.in_src.astype(np.int64)
        neigh = [set() for _ in range(n)]
        for u, v in zip(src.tolist(), dst.tolist()):  # undirected view, antiparallel edges once
            neigh[u].add(v)
            neigh[v].add(u)
        cap = max((n * 115 + 100 * p - 1) // (100 * p), 1)
        for _ in range(10):
            size = [0] * p
            nxt = label.copy()
            for v in range(n):
                freq = [0] * p
                freq[label[v]] = 1
                for u in neigh[v]:
                    freq[label[u]] += 1
                best = p
                for c in range(p):
                    if size[c] >= cap:
                        continue
                    if best == p or freq[c] > freq[best]:
                        best = c
                nxt[v] = best
                size[best] += 1
            label = nxt
        size = np.bincount(label, minlength=p).tolist()
        for c in range(p):  # a starved label gets one node from the largest part (:95-110)
            if size[c] > 0:
                continue
            donor = int(np.argmax(size))
            for v in range(n - 1, -1, -1):
                if label[v] == donor:
                    label[v] = c
                    size[donor] -= 1
                    size[c] += 1
                    break
        a = label.astype(np.uint32)
    else:
        raise ValueError(method)
    base = [np.nonzero(a == i)[0].astype(np.uint32) for i in range(p)]
    return extend_partition_np(csr, Partitioning(p, 0, a, base, []), 0)


def extend_partition_np(csr: "Csr", part: Partitioning, h: int) -> Partitioning:
    """extend_partition, proj/src/partition.cpp:123-145: h-step in-neighbourhood closure."""
    ext = []
    off = csr.in_offsets.astype(np.int64)
    for i in range(part.p):
        mask = np.zeros(csr.n, dtype=np.uint8)
        frontier = part.base[i].astype(np.int64)
        mask[frontier] = 1
        for _ in range(h):
            if frontier.size == 0:
                break
            lens = off[frontier + 1] - off[frontier]
            idx = np.repeat(off[frontier], lens) + (np.arange(lens.sum()) -
                                                    np.repeat(np.cumsum(lens) - lens, lens))
            u = np.unique(csr.in_src[idx].astype(np.int64))
            u = u[mask[u] == 0]
            mask[u] = 1
            frontier = u
        ext.append(mask)
    return Partitioning(part.p, h, part.assign, part.base, ext)


def ranked_by_score(score) -> list:
    """ranked_by_score, evaluation.cpp:110-119: score descending, ties by ascending id."""
    score = np.asarray(score, dtype=np.float64)
    return [int(x) for x in np.lexsort((np.arange(score.size), -score))]


def edges_into_nodes(off, weight, nodes, k) -> list:
    """edges_into_nodes, evaluation.cpp:121-151: the k heaviest in-edges of the ranked nodes,
    taken round-robin (per node: weight descending, ties by edge id)."""
    per_node = []
    for v in nodes:
        lo, hi = int(off[v]), int(off[v + 1])
        ids = np.arange(lo, hi)
        per_node.append([int(e) for e in ids[np.lexsort((ids, -np.asarray(weight[lo:hi])))]])
    out, nxt = [], [0] * len(nodes)
    while len(out) < k:
        advanced = False
        for i in range(len(nodes)):
            if len(out) >= k:
                break
            if nxt[i] < len(per_node[i]):
                out.append(per_node[i][nxt[i]])
                nxt[i] += 1
                advanced = True
        if not advanced:
            raise BuildError("not enough incoming edges among ranked nodes")
    return out


def part_quotas(total_target: int, sizes: list, n: int) -> list:
    """Largest-remainder quotas proportional to |part|, proj/src/partition.cpp:163-181."""
    targets, rema, assigned = [], [], 0
    for i, sz in enumerate(sizes):
        share = float(total_target) * float(sz) / float(n)
        t = int(share)
        targets.append(t)
        assigned += t
        rema.append((share - float(t), i))
    rema.sort(key=lambda a: (-a[0], a[1]))
    for r in range(total_target - assigned):
        targets[rema[r % len(sizes)][1]] += 1
    return targets


PART_STRIDE = 1 << 40  # worker-id window per part, proj/src/partition.cpp:14


class _OrcCfg(C.Structure):
    _fields_ = [("heuristic", C.c_int), ("window", C.c_uint32), ("batch_size", C.c_uint32),
                ("max_attempts", C.c_uint64)]


class _OrcSchedule(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("delta", C.c_double), ("lambda_", C.c_double),
                ("lambda1", C.c_double), ("n_max", C.c_double), ("k", C.c_uint32),
                ("t_max", C.c_uint32), ("lambda_samples", C.c_uint64)]


class _OrcResult(C.Structure):
    _fields_ = [("k", C.c_uint32), ("iterations", C.c_uint32), ("coverage", C.c_uint64),
                ("samples_used", C.c_uint64), ("attempts", C.c_uint64),
                ("est_suspension", C.c_double), ("passed_check", C.c_int)]


class _OrcSuspension(C.Structure):
    _fields_ = [("value", C.c_double), ("capped", C.c_int), ("runs", C.c_uint64)]


class _RefResult(C.Structure):
    _fields_ = [("k", C.c_uint32), ("iterations", C.c_uint32), ("coverage", C.c_uint64),
                ("samples_used", C.c_uint64), ("attempts", C.c_uint64),
                ("est_suspension", C.c_double), ("wall_time_s", C.c_double),
                ("passed_check", C.c_int)]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"status {status}: {msg}")
        self.status = status


def _sets(set_off, items):
    set_off = np.ascontiguousarray(set_off, dtype=np.uint64)
    items = np.ascontiguousarray(items, dtype=np.uint32)
    if items.size == 0:
        items = np.zeros(1, dtype=np.uint32)
    return set_off, items


def _cand(cand):
    if cand is None:
        return None, 0, 0
    a = np.ascontiguousarray(cand, dtype=np.uint32)
    if a.size == 0:
        return np.zeros(1, dtype=np.uint32), 0, 1
    return a, a.size, 1


class Port:
    """Plain-C restatement (kind = 'port')."""

    kind = "port"

    def __init__(self):
        build()
        L = self.L = C.CDLL(PORT_SO)
        L.orc_prg_next.restype = C.c_uint64
        L.orc_u01.restype = C.c_double
        L.orc_u01.argtypes = [C.c_uint64]
        L.orc_seed_from_worker.restype = C.c_uint64
        L.orc_seed_from_worker.argtypes = [C.c_uint64]
        L.orc_pick_uniform_node.restype = C.c_uint32
        L.orc_splitmix_next.argtypes = [C.c_uint64, u64p, u64p]
        L.orc_thread_sample.restype = C.c_uint32
        L.orc_thread_sample.argtypes = [C.POINTER(_OrcGraph), C.c_uint64, C.c_uint32,
                                        C.POINTER(_OrcCfg), u64p, u32p, u64p]
        L.orc_decode.argtypes = [C.POINTER(_OrcGraph), C.c_uint64, C.c_uint32, u32p, C.c_uint32,
                                 u32p, u32p]
        L.orc_stream_samples.argtypes = [C.POINTER(_OrcGraph), C.c_uint64, C.c_uint64,
                                         C.POINTER(_OrcCfg), C.POINTER(C.c_void_p)]
        L.orc_part_sample.argtypes = [C.POINTER(_OrcGraph), C.c_uint64, C.c_uint64,
                                      C.POINTER(_OrcCfg), C.POINTER(C.c_void_p), u64p, u64p]
        L.orc_rr_node_sets.argtypes = [C.POINTER(_OrcGraph), u64p, C.c_uint32, u64p, u32p,
                                       C.c_uint64]
        L.orc_pool_stats.argtypes = [C.c_void_p, u64p, u64p, u64p]
        L.orc_pool_copy.argtypes = [C.c_void_p, u64p, u32p, u32p, u64p, u32p]
        L.orc_pool_free.argtypes = [C.c_void_p]
        L.orc_greedy.argtypes = [C.c_uint32, C.c_uint64, u64p, u32p, u32p, C.c_uint64, C.c_uint32,
                                 C.c_int, u32p, u64p]
        L.orc_coverage_of.argtypes = [C.c_uint32, C.c_uint64, u64p, u32p, u32p, C.c_uint64, u32p,
                                      C.c_uint64, u64p]
        L.orc_ln_choose.restype = C.c_double
        L.orc_ln_choose.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_schedule_m.argtypes = [C.c_uint64, C.c_uint32, C.c_double, C.c_double,
                                     C.POINTER(_OrcSchedule)]
        L.orc_check.argtypes = [C.c_double, C.c_double, C.c_double, C.POINTER(_OrcSchedule),
                                C.c_uint32, f64p]
        L.orc_interdict.argtypes = [C.POINTER(_OrcGraph), C.c_int, u32p, C.c_uint64, C.c_uint32,
                                    C.c_double, C.c_double, C.c_uint64, C.POINTER(_OrcCfg),
                                    C.POINTER(_OrcResult), u32p]
        L.orc_lt_forward_simulate.restype = C.c_uint32
        L.orc_lt_forward_simulate.argtypes = [C.POINTER(_OrcGraph), u64p]
        L.orc_paired_runs.argtypes = [C.POINTER(_OrcGraph), C.c_int, u32p, C.c_uint64, u64p,
                                      C.c_uint64, u32p, u32p]
        L.orc_estimate_suspension.argtypes = [C.POINTER(_OrcGraph), C.c_int, u32p, C.c_uint64,
                                              C.c_double, C.c_double, u64p,
                                              C.POINTER(_OrcSuspension)]

    # -- prng
    def splitmix_next(self, state):
        a, b = C.c_uint64(), C.c_uint64()
        self.L.orc_splitmix_next(state, C.byref(a), C.byref(b))
        return a.value, b.value

    def prg_next(self, state):
        s = C.c_uint64(state)
        out = self.L.orc_prg_next(C.byref(s))
        return s.value, out

    def u01(self, out):
        return self.L.orc_u01(out)

    def seed_from_worker(self, w):
        return self.L.orc_seed_from_worker(w)

    def pick_uniform_node(self, state, n):
        s = C.c_uint64(state)
        v = self.L.orc_pick_uniform_node(C.byref(s), C.c_uint32(n))
        return s.value, v

    # -- helpers
    @staticmethod
    def _g(csr: Csr, domain=None, allowed=None):
        if domain is None:
            return _OrcGraph(csr.n, csr.m, _p(csr.in_offsets, u64p), _p(csr.in_src, u32p),
                             _p(csr.in_cum, f64p), _p(csr.p_of, f64p), None, 0, None)
        return _OrcGraph(csr.n, csr.m, _p(csr.in_offsets, u64p), _p(csr.in_src, u32p),
                         _p(csr.in_cum, f64p), _p(csr.p_of, f64p), _p(domain, u32p), domain.size,
                         allowed.ctypes.data_as(C.POINTER(C.c_uint8)))

    # -- ranking baselines (proj/src/evaluation.cpp:110-191,310-395)
    def rr_node_sets(self, csr, state, count):
        """-> (set_off u64[count + 1], items, state_after)"""
        g = self._g(csr)
        s = C.c_uint64(state)
        off = np.zeros(count + 1, dtype=np.uint64)
        cap = max(4096, count * 64)
        while True:
            items = np.zeros(cap, dtype=np.uint32)
            s = C.c_uint64(state)
            rc = self.L.orc_rr_node_sets(C.byref(g), C.byref(s), count, _p(off, u64p),
                                         _p(items, u32p), cap)
            if rc == 0:
                return off, items[: int(off[-1])].copy(), s.value
            cap *= 4

    def baseline(self, csr, weight, kind, mode, k, state, infmax_samples=100000):
        """baseline(), evaluation.cpp:330-395 -> (ids, state_after). kind: 'pagerank', 'maxdegree',
        'randomized', 'infmax-v', 'infmax-vi'; mode 0 edge / 1 node; weight = ProbGraph::weight."""
        n, m = csr.n, csr.m
        off = csr.in_offsets.astype(np.int64)
        if kind == "randomized":  # distinct_uniform, :153-165
            limit, seen, out, s = (m if mode == 0 else n), set(), [], state
            if k > limit:
                raise BuildError("k exceeds candidate count")
            while len(out) < k:
                s, o = self.prg_next(s)
                x = int(self.u01(o) * limit)
                x = min(x, limit - 1)
                if x not in seen:
                    seen.add(x)
                    out.append(x)
            return out, s
        in_deg = np.diff(off)
        out_deg = np.bincount(csr.in_src, minlength=n).astype(np.int64)
        dst = np.repeat(np.arange(n, dtype=np.int64), in_deg)
        if kind == "pagerank":  # pagerank_scores, :310-328 (sequential accumulation order)
            pr = np.full(n, 1.0 / n)
            for _ in range(200):
                dangling = 0.0
                for v in np.nonzero(out_deg == 0)[0]:
                    dangling += pr[v]
                base = (1.0 - 0.85) / n + 0.85 * dangling / n
                nxt = np.full(n, base)
                contrib = 0.85 * pr[csr.in_src] / out_deg[csr.in_src]
                for e in range(m):
                    nxt[dst[e]] += contrib[e]
                diff = 0.0
                for v in range(n):
                    diff += abs(nxt[v] - pr[v])
                pr = nxt
                if diff < 1e-10:
                    break
            ranked = ranked_by_score(pr)
        elif kind == "maxdegree":
            ranked = ranked_by_score((out_deg + in_deg).astype(np.float64))
        else:
            so, items, state = self.rr_node_sets(csr, state, infmax_samples)
            if kind == "infmax-vi":
                cand = np.nonzero(csr.p_of > 0)[0].astype(np.uint32)
                if cand.size == 0:
                    raise BuildError("suspect set is empty")
                ncand = cand.size
            else:
                cand, ncand = None, n
            budget = min(ncand, max(k, 64) if mode == 0 else k)
            sol, _ = self.greedy(n, so, items, budget, cand=cand, kind=1)
            ranked = [int(x) for x in sol]
        ranked = [int(x) for x in ranked]
        if mode == 1:
            if k > len(ranked):
                raise BuildError("k exceeds candidate count")
            return ranked[:k], state
        if k > m:
            raise BuildError("k exceeds edge count")
        listed = np.zeros(n, dtype=bool)
        listed[ranked] = True
        ranked += [int(v) for v in np.nonzero(~listed)[0]]
        return edges_into_nodes(off, weight, ranked, k), state

    # -- partitioned sampling (proj/src/partition.cpp:153-279)
    def distributed_sample(self, csr, part: "Partitioning", total_target, seed=0, heuristic=0,
                           window=2, batch_size=10, max_attempts=100_000_000) -> "DistributedData":
        for i in range(part.p):
            if part.base[i].size == 0:
                raise BuildError(f"part {i} is empty")
        targets = part_quotas(total_target, [b.size for b in part.base], csr.n)
        cfg = self._cfg(heuristic, window, batch_size, max_attempts)
        pools, crossings, attempts = [], 0, 0
        M = (1 << 64) - 1
        for i in range(part.p):
            dom = np.ascontiguousarray(part.base[i], dtype=np.uint32)
            mask = np.ascontiguousarray(part.extended[i], dtype=np.uint8)
            g = self._g(csr, dom, mask)
            h, cr, at = C.c_void_p(), C.c_uint64(), C.c_uint64()
            rc = self.L.orc_part_sample(C.byref(g), targets[i], (seed + i * PART_STRIDE) & M,
                                        C.byref(cfg), C.byref(h), C.byref(cr), C.byref(at))
            if rc:
                raise OracleError(rc, "distributed_sample")
            try:
                pools.append(_copy_pool(self.L.orc_pool_stats, self.L.orc_pool_copy, h))
            finally:
                self.L.orc_pool_free(h)
            crossings += cr.value
            attempts += at.value
        return DistributedData(concat_pools(pools, attempts), crossings, attempts,
                               crossings / attempts if attempts else 0.0, targets)

    @staticmethod
    def _cfg(heuristic=0, window=2, batch_size=10, max_attempts=100_000_000):
        return _OrcCfg(heuristic, window, batch_size, max_attempts)

    # -- sampler
    def thread_sample(self, csr, worker_id, l, heuristic=0, window=2, want_stats=False):
        g, cfg = self._g(csr), self._cfg(heuristic, window)
        seeds = np.zeros(max(l, 1), dtype=np.uint64)
        lens = np.zeros(max(l, 1), dtype=np.uint32)
        stats = np.zeros(4, dtype=np.uint64)
        cnt = self.L.orc_thread_sample(C.byref(g), worker_id, l, C.byref(cfg), _p(seeds, u64p),
                                       _p(lens, u32p), _p(stats, u64p))
        if want_stats:
            return seeds[:cnt].copy(), lens[:cnt].copy(), stats
        return seeds[:cnt].copy(), lens[:cnt].copy()

    def decode(self, csr, seed, length):
        g = self._g(csr)
        mark = np.zeros(max(csr.n, 1), dtype=np.uint32)
        nodes = np.zeros(length + 2, dtype=np.uint32)
        edges = np.zeros(length + 1, dtype=np.uint32)
        rc = self.L.orc_decode(C.byref(g), seed, length, _p(mark, u32p), 1, _p(nodes, u32p),
                               _p(edges, u32p))
        if rc < 0:
            raise OracleError(-rc, "decode")
        if rc == 0:
            return None
        return nodes[: length + 1].copy(), edges[:length].copy()

    def stream_samples(self, csr, target, seed=0, workers=1, heuristic=0, window=2, batch_size=10,
                       max_attempts=100_000_000) -> PoolData:
        g, cfg = self._g(csr), self._cfg(heuristic, window, batch_size, max_attempts)
        h = C.c_void_p()
        rc = self.L.orc_stream_samples(C.byref(g), target, seed, C.byref(cfg), C.byref(h))
        if rc:
            raise OracleError(rc, "stream_samples")
        try:
            return _copy_pool(self.L.orc_pool_stats, self.L.orc_pool_copy, h)
        finally:
            self.L.orc_pool_free(h)

    # -- coverage
    def greedy(self, limit, set_off, items, k, cand=None, lazy=True, kind=0):
        set_off, items = _sets(set_off, items)
        ca, nc, _ = _cand(cand)
        sol = np.zeros(max(k, 1), dtype=np.uint32)
        cov = C.c_uint64()
        rc = self.L.orc_greedy(limit, len(set_off) - 1, _p(set_off, u64p), _p(items, u32p),
                               _p(ca, u32p), nc, k, int(lazy), _p(sol, u32p), C.byref(cov))
        if rc:
            raise OracleError(rc, "greedy")
        return sol[:k].copy(), cov.value

    def coverage_of(self, limit, set_off, items, query, cand=None, kind=0):
        set_off, items = _sets(set_off, items)
        ca, nc, _ = _cand(cand)
        q = np.ascontiguousarray(query, dtype=np.uint32)
        cov = C.c_uint64()
        rc = self.L.orc_coverage_of(limit, len(set_off) - 1, _p(set_off, u64p), _p(items, u32p),
                                    _p(ca, u32p), nc, _p(q, u32p), q.size, C.byref(cov))
        if rc:
            raise OracleError(rc, "coverage_of")
        return cov.value

    def ln_choose(self, M, k):
        return self.L.orc_ln_choose(M, k)

    def schedule(self, M, k, eps, delta):
        s = _OrcSchedule()
        rc = self.L.orc_schedule_m(M, k, eps, delta, C.byref(s))
        if rc:
            raise OracleError(rc, "schedule")
        return dict(n_max=s.n_max, lambda_=s.lambda_, lambda1=s.lambda1, t_max=s.t_max,
                    lambda_samples=s.lambda_samples)

    def check(self, cov_r, cov_rp, n_rp, M, k, eps, delta, t):
        s = _OrcSchedule()
        rc = self.L.orc_schedule_m(M, k, eps, delta, C.byref(s))
        if rc:
            raise OracleError(rc, "schedule")
        e = C.c_double()
        ok = self.L.orc_check(float(cov_r), float(cov_rp), float(n_rp), C.byref(s), t, C.byref(e))
        return bool(ok), e.value

    def interdict(self, csr, kind, k, eps, delta, seed=0, cand=None, workers=1, batch_size=10,
                  max_attempts=100_000_000):
        g, cfg = self._g(csr), self._cfg(0, 2, batch_size, max_attempts)
        ca, nc, has = _cand(cand)
        res = _OrcResult()
        sol = np.zeros(max(k, 1), dtype=np.uint32)
        rc = self.L.orc_interdict(C.byref(g), kind, _p(ca, u32p) if has else None, nc, k, eps,
                                  delta, seed, C.byref(cfg), C.byref(res), _p(sol, u32p))
        if rc:
            raise OracleError(rc, "interdict")
        return dict(kind="edge" if kind == 0 else "node", k=res.k, epsilon=eps, delta=delta,
                    solution=[int(x) for x in sol[:k]], est_suspension=res.est_suspension,
                    coverage=res.coverage, samples_used=res.samples_used, attempts=res.attempts,
                    iterations=res.iterations, passed_check=bool(res.passed_check))

    # -- paired LT forward simulation (proj/src/evaluation.cpp:49-108,202-242)
    def lt_forward_simulate(self, csr, state):
        """-> (infected, state_after)"""
        g = self._g(csr)
        s = C.c_uint64(state)
        r = self.L.orc_lt_forward_simulate(C.byref(g), C.byref(s))
        return int(r), s.value

    def paired_runs(self, csr, kind, ids, state, nruns):
        """-> (full u32[nruns], residual u32[nruns], state_after)"""
        g = self._g(csr)
        a = np.ascontiguousarray(ids, dtype=np.uint32)
        buf = a if a.size else np.zeros(1, dtype=np.uint32)
        full = np.zeros(max(nruns, 1), dtype=np.uint32)
        res = np.zeros(max(nruns, 1), dtype=np.uint32)
        s = C.c_uint64(state)
        rc = self.L.orc_paired_runs(C.byref(g), kind, _p(buf, u32p), a.size, C.byref(s), nruns,
                                    _p(full, u32p), _p(res, u32p))
        if rc:
            raise OracleError(rc, "paired_runs")
        return full[:nruns], res[:nruns], s.value

    def estimate_suspension(self, csr, kind, ids, eps, delta, state):
        """-> dict(value, capped, runs, state)"""
        g = self._g(csr)
        a = np.ascontiguousarray(ids, dtype=np.uint32)
        buf = a if a.size else np.zeros(1, dtype=np.uint32)
        s = C.c_uint64(state)
        out = _OrcSuspension()
        rc = self.L.orc_estimate_suspension(C.byref(g), kind, _p(buf, u32p), a.size, eps, delta,
                                            C.byref(s), C.byref(out))
        if rc:
            raise OracleError(rc, "estimate_suspension")
        return dict(value=out.value, capped=bool(out.capped), runs=int(out.runs), state=s.value)


def concat_pools(pools, attempts) -> "PoolData":
    """Pools of the parts appended in part order (partition.cpp:263-266)."""
    eo, base = [np.zeros(1, dtype=np.uint64)], 0
    for q in pools:
        eo.append(q.edge_off[1:].astype(np.uint64) + np.uint64(base))
        base += int(q.edge_off[-1])
    cat = lambda xs, dt: np.concatenate(xs) if xs else np.zeros(0, dtype=dt)
    return PoolData(attempts, np.concatenate(eo), cat([q.nodes for q in pools], np.uint32),
                    cat([q.edges for q in pools], np.uint32),
                    cat([q.tag_worker for q in pools], np.uint64),
                    cat([q.tag_seq for q in pools], np.uint32))


def _copy_pool(stats_fn, copy_fn, h) -> PoolData:
    ns, at, te = C.c_uint64(), C.c_uint64(), C.c_uint64()
    stats_fn(h, C.byref(ns), C.byref(at), C.byref(te))
    ns, at, te = ns.value, at.value, te.value
    eo = np.zeros(ns + 1, dtype=np.uint64)
    nodes = np.zeros(max(te + ns, 1), dtype=np.uint32)
    edges = np.zeros(max(te, 1), dtype=np.uint32)
    tw = np.zeros(max(ns, 1), dtype=np.uint64)
    ts = np.zeros(max(ns, 1), dtype=np.uint32)
    copy_fn(h, _p(eo, u64p), _p(nodes, u32p), _p(edges, u32p), _p(tw, u64p), _p(ts, u32p))
    return PoolData(at, eo, nodes[: te + ns], edges[:te], tw[:ns], ts[:ns])


class Ref:
    """The unmodified reference library through ref_shim.cpp (kind = 'reference')."""

    kind = "reference"

    def __init__(self):
        build()
        if not have_ref():
            raise FileNotFoundError(REF_SO)
        L = self.L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_prg_next.restype = C.c_uint64
        L.ref_u01.restype = C.c_double
        L.ref_u01.argtypes = [C.c_uint64]
        L.ref_seed_from_worker.restype = C.c_uint64
        L.ref_seed_from_worker.argtypes = [C.c_uint64]
        L.ref_pick_uniform_node.restype = C.c_uint32
        L.ref_splitmix_next.argtypes = [C.c_uint64, u64p, u64p]
        L.ref_graph_from_csr.restype = C.c_void_p
        L.ref_graph_from_csr.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f64p]
        L.ref_baseline.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_uint32, u64p,
                                   C.c_uint32, u32p]
        L.ref_partition_graph.argtypes = [C.c_void_p, C.c_uint32, C.c_int, C.c_uint64, u32p,
                                          C.POINTER(C.c_void_p)]
        L.ref_extend_partition.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32,
                                           C.POINTER(C.c_void_p)]
        L.ref_partition_copy.argtypes = [C.c_void_p, u32p, C.POINTER(C.c_uint8)]
        L.ref_partition_copy.restype = None
        L.ref_partition_free.argtypes = [C.c_void_p]
        L.ref_partition_free.restype = None
        L.ref_distributed_sample.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                             C.c_uint64, C.c_uint32, C.c_int, C.c_uint32,
                                             C.c_uint32, C.c_uint64, C.POINTER(C.c_void_p), u64p,
                                             u64p, f64p, u64p]
        L.ref_graph_from_csr_lean.restype = C.c_void_p
        L.ref_graph_from_csr_lean.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f64p]
        L.ref_graph_build.argtypes = [C.c_uint32, C.c_uint64, u32p, u32p, f64p, C.c_int,
                                      C.c_uint64, C.POINTER(C.c_void_p)]
        L.ref_graph_load_edge_list.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.c_int,
                                               C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_graph_synth.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(C.c_void_p)]
        L.ref_graph_save_cache.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_graph_load_cache.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_graph_save_edge_list.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_graph_validate.argtypes = [C.c_void_p]
        L.ref_graph_dims.argtypes = [C.c_void_p, u32p, u32p]
        L.ref_graph_copy.argtypes = [C.c_void_p, u64p, u32p, f64p, f64p, u32p]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_suspects_from_p.argtypes = [C.c_void_p, f64p, C.POINTER(C.c_void_p)]
        L.ref_suspects_random.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64,
                                          C.POINTER(C.c_void_p)]
        L.ref_suspects_load.argtypes = [C.c_char_p, C.c_void_p, C.POINTER(C.c_void_p)]
        L.ref_suspects_copy_p.argtypes = [C.c_void_p, f64p]
        L.ref_suspects_size.restype = C.c_uint64
        L.ref_suspects_size.argtypes = [C.c_void_p]
        L.ref_suspects_free.argtypes = [C.c_void_p]
        L.ref_thread_sample.restype = C.c_int64
        L.ref_thread_sample.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_int,
                                        C.c_uint32, u64p, u32p]
        L.ref_decode.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, u32p, u32p]
        L.ref_stream_samples.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64,
                                         C.c_uint64, C.c_int, C.c_uint32, C.c_uint32, C.c_uint64,
                                         C.POINTER(C.c_void_p)]
        L.ref_pool_stats.argtypes = [C.c_void_p, u64p, u64p, u64p]
        L.ref_pool_copy.argtypes = [C.c_void_p, u64p, u32p, u32p, u64p, u32p]
        L.ref_pool_free.argtypes = [C.c_void_p]
        L.ref_greedy.argtypes = [C.c_int, C.c_uint32, C.c_uint64, u64p, u32p, u32p, C.c_uint64,
                                 C.c_int, C.c_uint32, C.c_int, u32p, u64p]
        L.ref_coverage_of.argtypes = [C.c_int, C.c_uint32, C.c_uint64, u64p, u32p, u32p,
                                      C.c_uint64, C.c_int, u32p, C.c_uint64, u64p]
        L.ref_schedule.argtypes = [C.c_uint64, C.c_uint32, C.c_double, C.c_double, f64p, u32p]
        L.ref_ln_choose.restype = C.c_double
        L.ref_ln_choose.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_check_solution.argtypes = [C.c_int, C.c_uint32, C.c_uint64, u64p, u32p, C.c_uint64,
                                         u64p, u32p, u32p, C.c_uint64, C.c_int, u32p, C.c_uint64,
                                         C.c_uint64, C.c_uint32, C.c_double, C.c_double,
                                         C.c_uint32, C.POINTER(C.c_int), f64p]
        L.ref_interdict.argtypes = [C.c_void_p, C.c_void_p, C.c_int, u32p, C.c_uint64, C.c_int,
                                    C.c_uint32, C.c_double, C.c_double, C.c_uint32, C.c_uint64,
                                    C.c_uint32, C.c_uint64, C.POINTER(_RefResult), u32p,
                                    C.c_char_p, C.c_uint64]

        L.ref_lt_forward_simulate.argtypes = [C.c_void_p, C.c_void_p, u64p, u32p]
        L.ref_estimate_suspension.argtypes = [C.c_void_p, C.c_void_p, C.c_int, u32p, C.c_uint64,
                                              C.c_double, C.c_double, u64p, f64p,
                                              C.POINTER(C.c_int), u64p]

    def _chk(self, rc, what):
        if rc:
            raise OracleError(rc, f"{what}: {self.L.ref_last_error().decode()}")

    # -- prng
    def splitmix_next(self, state):
        a, b = C.c_uint64(), C.c_uint64()
        self.L.ref_splitmix_next(state, C.byref(a), C.byref(b))
        return a.value, b.value

    def prg_next(self, state):
        s = C.c_uint64(state)
        out = self.L.ref_prg_next(C.byref(s))
        return s.value, out

    def u01(self, out):
        return self.L.ref_u01(out)

    def seed_from_worker(self, w):
        return self.L.ref_seed_from_worker(w)

    def pick_uniform_node(self, state, n):
        s = C.c_uint64(state)
        v = self.L.ref_pick_uniform_node(C.byref(s), C.c_uint32(n))
        return s.value, v

    # -- graph handles -> Csr
    def _to_csr(self, gh, p_of=None) -> Csr:
        n, m = C.c_uint32(), C.c_uint32()
        self.L.ref_graph_dims(gh, C.byref(n), C.byref(m))
        n, m = n.value, m.value
        off = np.zeros(n + 1, dtype=np.uint64)
        src = np.zeros(max(m, 1), dtype=np.uint32)
        cum = np.zeros(max(m, 1), dtype=np.float64)
        self.L.ref_graph_copy(gh, _p(off, u64p), _p(src, u32p), _p(cum, f64p), None, None)
        return Csr(n, m, off, src[:m], cum[:m], np.zeros(n) if p_of is None else p_of)

    def graph_extra(self, gh):
        """(weight f64[m], edge_dst u32[m]) of a graph handle."""
        n, m = C.c_uint32(), C.c_uint32()
        self.L.ref_graph_dims(gh, C.byref(n), C.byref(m))
        w = np.zeros(max(m.value, 1), dtype=np.float64)
        d = np.zeros(max(m.value, 1), dtype=np.uint32)
        self.L.ref_graph_copy(gh, None, None, None, _p(w, f64p), _p(d, u32p))
        return w[: m.value], d[: m.value]

    def build_graph(self, n, u, v, w=None, mode=1, seed=0):
        u = np.ascontiguousarray(u, dtype=np.uint32)
        v = np.ascontiguousarray(v, dtype=np.uint32)
        wa = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
        h = C.c_void_p()
        self._chk(self.L.ref_graph_build(n, u.size, _p(u, u32p), _p(v, u32p), _p(wa, f64p), mode,
                                         seed, C.byref(h)), "build_graph")
        return h

    def load_edge_list(self, path, mode=1, seed=0, symmetrize=False, mapping_out=None):
        h = C.c_void_p()
        self._chk(self.L.ref_graph_load_edge_list(
            path.encode(), mode, seed, int(symmetrize),
            mapping_out.encode() if mapping_out else None, C.byref(h)), "load_edge_list")
        return h

    def synth_graph(self, n, density, seed):
        h = C.c_void_p()
        self._chk(self.L.ref_graph_synth(n, density, seed, C.byref(h)), "synth_graph")
        return h

    def graph_from_csr(self, csr: Csr):
        return C.c_void_p(self.L.ref_graph_from_csr(csr.n, csr.m, _p(csr.in_offsets, u64p),
                                                    _p(csr.in_src, u32p), _p(csr.in_cum, f64p)))

    def save_cache(self, gh, path):
        self._chk(self.L.ref_graph_save_cache(gh, path.encode()), "save_cache")

    def load_cache(self, path):
        h = C.c_void_p()
        self._chk(self.L.ref_graph_load_cache(path.encode(), C.byref(h)), "load_cache")
        return h

    def save_edge_list(self, gh, path):
        self._chk(self.L.ref_graph_save_edge_list(gh, path.encode()), "save_edge_list")

    def validate(self, gh):
        self._chk(self.L.ref_graph_validate(gh), "validate")

    def graph_free(self, gh):
        self.L.ref_graph_free(gh)

    def random_suspects(self, gh, count, seed) -> np.ndarray:
        h = C.c_void_p()
        self._chk(self.L.ref_suspects_random(gh, count, seed, C.byref(h)), "random_suspects")
        return self._p_of(gh, h)

    def load_suspects(self, path, gh) -> np.ndarray:
        h = C.c_void_p()
        self._chk(self.L.ref_suspects_load(path.encode(), gh, C.byref(h)), "load_suspects")
        return self._p_of(gh, h)

    def _p_of(self, gh, vh):
        n, m = C.c_uint32(), C.c_uint32()
        self.L.ref_graph_dims(gh, C.byref(n), C.byref(m))
        p = np.zeros(max(n.value, 1), dtype=np.float64)
        self.L.ref_suspects_copy_p(vh, _p(p, f64p))
        self.L.ref_suspects_free(vh)
        return p[: n.value]

    class _Handles:
        def __init__(self, ref, csr, lean=False):
            self.ref = ref
            if lean:  # sampler-only ProbGraph (no weight / edge_dst): the 10^9-edge bench shapes
                self.g = C.c_void_p(ref.L.ref_graph_from_csr_lean(
                    csr.n, csr.m, _p(csr.in_offsets, u64p), _p(csr.in_src, u32p),
                    _p(csr.in_cum, f64p)))
            else:
                self.g = ref.graph_from_csr(csr)
            self.vi = C.c_void_p()
            ref._chk(ref.L.ref_suspects_from_p(self.g, _p(csr.p_of, f64p), C.byref(self.vi)),
                     "suspects")

        def __enter__(self):
            return self

        def __exit__(self, *a):
            self.ref.L.ref_suspects_free(self.vi)
            self.ref.L.ref_graph_free(self.g)

    def handles(self, csr: Csr, lean=False):
        return Ref._Handles(self, csr, lean)

    BASELINES = {"pagerank": 0, "maxdegree": 1, "randomized": 2, "infmax-v": 3, "infmax-vi": 4}

    def baseline(self, csr, kind, mode, k, state, infmax_samples=100000, hd=None):
        """baseline() by the reference -> (ids, state_after)."""
        ids = np.zeros(max(k, 1), dtype=np.uint32)

        def run(h):
            s = C.c_uint64(state)
            self._chk(self.L.ref_baseline(h.g, h.vi, self.BASELINES[kind], mode, k, C.byref(s),
                                          infmax_samples, _p(ids, u32p)), "baseline")
            return [int(x) for x in ids[:k]], s.value

        if hd is not None:
            return run(hd)
        with self.handles(csr) as h:
            return run(h)

    # -- partitioned sampling (proj/include/hsaw/partition.hpp)
    def partition(self, csr, p, method="hash", seed=0, assign=None, hops=0, hd=None) -> "Partitioning":
        """partition_graph + extend_partition(h) by the reference -> Partitioning (numpy copy)."""
        code = {"hash": 0, "labelprop": 1, "external": 2}[method]
        a = None if assign is None else np.ascontiguousarray(assign, dtype=np.uint32)

        def run(h):
            ph, eh = C.c_void_p(), C.c_void_p()
            self._chk(self.L.ref_partition_graph(h.g, p, code, seed, _p(a, u32p), C.byref(ph)),
                      "partition_graph")
            try:
                self._chk(self.L.ref_extend_partition(h.g, ph, hops, C.byref(eh)), "extend_partition")
                try:
                    asg = np.zeros(csr.n, dtype=np.uint32)
                    ext = np.zeros((p, csr.n), dtype=np.uint8)
                    self.L.ref_partition_copy(eh, _p(asg, u32p),
                                              ext.ctypes.data_as(C.POINTER(C.c_uint8)))
                finally:
                    self.L.ref_partition_free(eh)
            finally:
                self.L.ref_partition_free(ph)
            base = [np.nonzero(asg == i)[0].astype(np.uint32) for i in range(p)]
            return Partitioning(p, hops, asg, base, [ext[i].copy() for i in range(p)])

        if hd is not None:
            return run(hd)
        with self.handles(csr) as h:
            return run(h)

    def distributed_sample(self, csr, part: "Partitioning", total_target, seed=0, workers=1,
                           heuristic=0, window=2, batch_size=10, max_attempts=100_000_000,
                           hd=None) -> "DistributedData":
        def run(h):
            ph, eh, pool = C.c_void_p(), C.c_void_p(), C.c_void_p()
            a = np.ascontiguousarray(part.assign, dtype=np.uint32)
            self._chk(self.L.ref_partition_graph(h.g, part.p, 2, 0, _p(a, u32p), C.byref(ph)),
                      "partition_graph")
            try:
                self._chk(self.L.ref_extend_partition(h.g, ph, part.hops, C.byref(eh)),
                          "extend_partition")
                try:
                    cr, at, fr = C.c_uint64(), C.c_uint64(), C.c_double()
                    tg = np.zeros(part.p, dtype=np.uint64)
                    self._chk(self.L.ref_distributed_sample(
                        h.g, h.vi, eh, total_target, seed, workers, heuristic, window, batch_size,
                        max_attempts, C.byref(pool), C.byref(cr), C.byref(at), C.byref(fr),
                        _p(tg, u64p)), "distributed_sample")
                    try:
                        pd = _copy_pool(self.L.ref_pool_stats, self.L.ref_pool_copy, pool)
                    finally:
                        self.L.ref_pool_free(pool)
                    return DistributedData(pd, cr.value, at.value, fr.value,
                                           [int(x) for x in tg])
                finally:
                    self.L.ref_partition_free(eh)
            finally:
                self.L.ref_partition_free(ph)

        if hd is not None:
            return run(hd)
        with self.handles(csr) as h:
            return run(h)

    # -- sampler (same signatures as Port)
    def thread_sample(self, csr, worker_id, l, heuristic=0, window=2, hd=None):
        seeds = np.zeros(max(l, 1), dtype=np.uint64)
        lens = np.zeros(max(l, 1), dtype=np.uint32)

        def run(h):
            cnt = self.L.ref_thread_sample(h.g, h.vi, worker_id, l, heuristic, window,
                                           _p(seeds, u64p), _p(lens, u32p))
            if cnt < 0:
                raise OracleError(-cnt, "thread_sample")
            return seeds[:cnt].copy(), lens[:cnt].copy()

        if hd is not None:
            return run(hd)
        with self.handles(csr) as h:
            return run(h)

    def decode(self, csr, seed, length, hd=None):
        nodes = np.zeros(length + 2, dtype=np.uint32)
        edges = np.zeros(length + 1, dtype=np.uint32)

        def run(h):
            rc = self.L.ref_decode(h.g, h.vi, seed, length, _p(nodes, u32p), _p(edges, u32p))
            if rc < 0:
                raise OracleError(-rc, "decode: " + self.L.ref_last_error().decode())
            return None if rc == 0 else (nodes[: length + 1].copy(), edges[:length].copy())

        if hd is not None:
            return run(hd)
        with self.handles(csr) as h:
            return run(h)

    def stream_samples(self, csr, target, seed=0, workers=1, heuristic=0, window=2, batch_size=10,
                       max_attempts=100_000_000, hd=None, copy=True):
        def run(h):
            ph = C.c_void_p()
            self._chk(self.L.ref_stream_samples(h.g, h.vi, workers, target, seed, heuristic,
                                                window, batch_size, max_attempts, C.byref(ph)),
                      "stream_samples")
            try:
                if copy:
                    return _copy_pool(self.L.ref_pool_stats, self.L.ref_pool_copy, ph)
                ns, at, te = C.c_uint64(), C.c_uint64(), C.c_uint64()
                self.L.ref_pool_stats(ph, C.byref(ns), C.byref(at), C.byref(te))
                return ns.value, at.value, te.value
            finally:
                self.L.ref_pool_free(ph)

        if hd is not None:
            return run(hd)
        with self.handles(csr) as h:
            return run(h)

    # -- coverage
    def greedy(self, limit, set_off, items, k, cand=None, lazy=True, kind=0):
        set_off, items = _sets(set_off, items)
        ca, nc, has = _cand(cand)
        sol = np.zeros(max(k, 1), dtype=np.uint32)
        cov = C.c_uint64()
        self._chk(self.L.ref_greedy(kind, limit, len(set_off) - 1, _p(set_off, u64p),
                                    _p(items, u32p), _p(ca, u32p), nc, has, k, int(not lazy),
                                    _p(sol, u32p), C.byref(cov)), "greedy")
        return sol[:k].copy(), cov.value

    def coverage_of(self, limit, set_off, items, query, cand=None, kind=0):
        set_off, items = _sets(set_off, items)
        ca, nc, has = _cand(cand)
        q = np.ascontiguousarray(query, dtype=np.uint32)
        cov = C.c_uint64()
        self._chk(self.L.ref_coverage_of(kind, limit, len(set_off) - 1, _p(set_off, u64p),
                                         _p(items, u32p), _p(ca, u32p), nc, has, _p(q, u32p),
                                         q.size, C.byref(cov)), "coverage_of")
        return cov.value

    def ln_choose(self, M, k):
        return self.L.ref_ln_choose(M, k)

    def schedule(self, M, k, eps, delta):
        out = np.zeros(4, dtype=np.float64)
        t = C.c_uint32()
        self._chk(self.L.ref_schedule(M, k, eps, delta, _p(out, f64p), C.byref(t)), "schedule")
        return dict(n_max=out[0], lambda_=out[1], lambda1=out[2], t_max=t.value,
                    lambda_samples=int(out[3]))

    def check_solution(self, limit, sets_r, sets_rp, solution, M, k, eps, delta, t, cand=None,
                       kind=0):
        so_r, it_r = _sets(*sets_r)
        so_p, it_p = _sets(*sets_rp)
        ca, nc, has = _cand(cand)
        sol = np.ascontiguousarray(solution, dtype=np.uint32)
        ok, e = C.c_int(), C.c_double()
        self._chk(self.L.ref_check_solution(kind, limit, len(so_r) - 1, _p(so_r, u64p),
                                            _p(it_r, u32p), len(so_p) - 1, _p(so_p, u64p),
                                            _p(it_p, u32p), _p(ca, u32p), nc, has, _p(sol, u32p),
                                            sol.size, M, k, eps, delta, t, C.byref(ok),
                                            C.byref(e)), "check_solution")
        return bool(ok.value), e.value

    def interdict(self, csr, kind, k, eps, delta, seed=0, cand=None, workers=1, batch_size=10,
                  max_attempts=100_000_000, hd=None, want_json=False):
        ca, nc, has = _cand(cand)
        res = _RefResult()
        sol = np.zeros(max(k, 1), dtype=np.uint32)
        buf = C.create_string_buffer(1 << 16)

        def run(h):
            self._chk(self.L.ref_interdict(h.g, h.vi, kind, _p(ca, u32p), nc, has, k, eps, delta,
                                           workers, seed, batch_size, max_attempts, C.byref(res),
                                           _p(sol, u32p), buf, len(buf)), "interdict")

        if hd is not None:
            run(hd)
        else:
            with self.handles(csr) as h:
                run(h)
        out = dict(kind="edge" if kind == 0 else "node", k=res.k, epsilon=eps, delta=delta,
                   solution=[int(x) for x in sol[:k]], est_suspension=res.est_suspension,
                   coverage=res.coverage, samples_used=res.samples_used, attempts=res.attempts,
                   iterations=res.iterations, passed_check=bool(res.passed_check))
        if want_json:
            out["json"] = buf.value.decode()
            out["wall_time_s"] = res.wall_time_s
        return out

    # -- paired LT forward simulation (proj/include/hsaw/evaluation.hpp:25-39)
    def lt_forward_simulate(self, csr, state, hd=None):
        def run(h):
            s, out = C.c_uint64(state), C.c_uint32()
            self._chk(self.L.ref_lt_forward_simulate(h.g, h.vi, C.byref(s), C.byref(out)),
                      "lt_forward_simulate")
            return int(out.value), s.value

        if hd is not None:
            return run(hd)
        with self.handles(csr) as h:
            return run(h)

    def estimate_suspension(self, csr, kind, ids, eps, delta, state, hd=None):
        a = np.ascontiguousarray(ids, dtype=np.uint32)
        buf = a if a.size else np.zeros(1, dtype=np.uint32)

        def run(h):
            s, v, cp, runs = C.c_uint64(state), C.c_double(), C.c_int(), C.c_uint64()
            self._chk(self.L.ref_estimate_suspension(h.g, h.vi, kind, _p(buf, u32p), a.size, eps,
                                                     delta, C.byref(s), C.byref(v), C.byref(cp),
                                                     C.byref(runs)), "estimate_suspension")
            return dict(value=v.value, capped=bool(cp.value), runs=int(runs.value), state=s.value)

        if hd is not None:
            return run(hd)
        with self.handles(csr) as h:
            return run(h)


# ---- build_graph restatement (numpy) ----------------------------------------------------------------
class BuildError(RuntimeError):
    """DataError of build_graph / validate (proj/src/graph.cpp:20), message as the reference's."""


def build_graph_np(n, u, v, w=None, mode=1):
    """Restatement of build_graph (proj/src/graph.cpp:112-199) + validate (:70-104) for
    WeightMode::Given (mode 0) and ::InDegree (mode 1): canonical (target, source) order, edge id =
    CSR position, per-row SEQUENTIAL float64 cumulative sums (np.add.accumulate adds left to right,
    like `cum += w`). Returns (in_offsets, in_src, in_cum, weight, edge_dst). Test infrastructure."""
    u = np.asarray(u, dtype=np.uint32)
    v = np.asarray(v, dtype=np.uint32)
    ne = u.size
    given = mode == 0
    wv = None if w is None else np.asarray(w, dtype=np.float64)
    for i in range(ne):  # graph.cpp:115-123, in input order
        a, b = int(u[i]), int(v[i])
        if a >= n or b >= n:
            raise BuildError("edge endpoint out of range")
        if a == b:
            raise BuildError(f"self-loop {a} -> {b}")
        if given and (not (wv[i] > 0.0) or wv[i] > 1.0):
            raise BuildError(f"weight {wv[i]:f} out of (0,1] on edge {a} -> {b}")
    order = np.lexsort((u, v))  # by target, then source (:125-128)
    su, sv = u[order], v[order]
    for i in range(1, ne):  # :129-134
        if su[i] == su[i - 1] and sv[i] == sv[i - 1]:
            raise BuildError(f"duplicate edge {int(su[i])} -> {int(sv[i])}")
    off = np.zeros(n + 1, dtype=np.uint64)
    np.add.at(off, sv.astype(np.int64) + 1, 1)
    off = np.cumsum(off).astype(np.uint64)
    cum = np.zeros(ne, dtype=np.float64)
    weight = np.zeros(ne, dtype=np.float64)
    sw = wv[order] if given else None
    for x in range(n):  # :149-193
        lo, hi = int(off[x]), int(off[x + 1])
        if hi == lo:
            continue
        weight[lo:hi] = sw[lo:hi] if given else 1.0 / float(hi - lo)
        cum[lo:hi] = np.add.accumulate(weight[lo:hi])
        if given and cum[hi - 1] > 1.0 + 1e-12:
            raise BuildError(f"in-weight sum {cum[hi - 1]:f} > 1 at node {x}")
    for x in range(n):  # validate(), :79-103
        lo, hi = int(off[x]), int(off[x + 1])
        prev = 0.0
        for i in range(lo, hi):
            if not (cum[i] > prev):
                raise BuildError(f"graph: cumulative weights not increasing at node {x}")
            prev = cum[i]
        if hi > lo and cum[hi - 1] > 1.0 + 1e-12:
            raise BuildError(f"graph: in-weight sum {cum[hi - 1]:f} > 1 at node {x}")
    return off, su.copy(), cum, weight, sv.copy()

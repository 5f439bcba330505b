"""Synthetic benchmark inputs: R-MAT graphs of the BASELINE.json shapes as reference-layout CSR.

Bench tooling, not part of the hot path. The reference only ships a uniform generator
(`synth_graph`, proj/src/graph.cpp:330-352); BASELINE.json asks for R-MAT shapes, so this module
builds them and hands the *same* arrays to the GPU path and to the CPU reference. The CSR follows
the reference's conventions exactly: in-edges grouped by target, sorted by source, edge id = CSR
slot (proj/include/hsaw/graph.hpp:15-18), LT weights 1/in-degree with the cumulative array formed
by *sequential* FP64 summation (proj/src/graph.cpp:169-180) — reproduced bit-exactly here because
np.add.accumulate is a strict left-to-right sum and every row of degree d shares one sequence.

The arrays bypass the reference's `validate()` on purpose: it rejects 1/d rows with d >= 36217
(rounding drift > 1e-12), which R-MAT hubs exceed; the sampler itself is well defined
on them (graph.hpp:66).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class CsrGraph:
    n: int
    m: int
    in_offsets: np.ndarray  # u64[n+1]
    in_src: np.ndarray      # u32[m]
    in_cum: np.ndarray      # f64[m]
    p_of: np.ndarray        # f64[n]

    @property
    def reference_bytes(self) -> int:
        """Sampler-visible bytes in the reference layout."""
        return 8 * (self.n + 1) + 12 * self.m + 8 * self.n


def indegree_cum(in_offsets: np.ndarray) -> np.ndarray:
    """in_cum for WeightMode::InDegree: per row, the sequential FP64 sum of d copies of 1.0/d."""
    deg = np.diff(in_offsets.astype(np.int64))
    m = int(in_offsets[-1])
    cum = np.empty(m, dtype=np.float64)
    order = np.argsort(deg, kind="stable")
    sdeg = deg[order]
    starts = in_offsets[:-1].astype(np.int64)[order]
    uniq, first = np.unique(sdeg, return_index=True)
    bounds = np.append(first, sdeg.size)
    for d, a, b in zip(uniq, bounds[:-1], bounds[1:]):
        d = int(d)
        if d == 0:
            continue
        seq = np.add.accumulate(np.full(d, 1.0 / float(d), dtype=np.float64))
        rows = starts[a:b]
        idx = (rows[:, None] + np.arange(d, dtype=np.int64)[None, :]).ravel()
        cum[idx] = np.tile(seq, rows.size)
    return cum


def csr_from_edges(n: int, u: np.ndarray, v: np.ndarray):
    """Canonical in-CSR (by target, then source) of distinct, loop-free directed edges u -> v."""
    key = v.astype(np.uint64) * np.uint64(n) + u.astype(np.uint64)
    key.sort()  # by (v, u); np.unique's hash path is ~6x slower than sort + adjacent compare
    if key.size:
        key = key[np.concatenate(([True], key[1:] != key[:-1]))]
    dst = (key // np.uint64(n)).astype(np.uint32)
    src = (key % np.uint64(n)).astype(np.uint32)
    keep = dst != src
    dst, src = dst[keep], src[keep]
    counts = np.bincount(dst, minlength=n).astype(np.uint64)
    off = np.zeros(n + 1, dtype=np.uint64)
    np.cumsum(counts, out=off[1:])
    return off, src


def random_suspects(n: int, count: int, seed: int) -> np.ndarray:
    """`count` distinct uniform nodes with p ~ U(0,1) (the shape of random_suspects,
    proj/src/graph.cpp:310-328; numpy's generator, not the reference stream)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    nodes = rng.choice(n, size=count, replace=False)
    p = rng.random(count)
    p[p == 0.0] = 0.5
    p_of = np.zeros(n, dtype=np.float64)
    p_of[nodes] = p
    return p_of


def rmat_graph(scale: int, edge_factor: float, seed: int = 1, abcd=(0.57, 0.19, 0.19, 0.05),
               suspect_frac: float = 0.01, suspect_seed: int = 2, n: int | None = None) -> CsrGraph:
    """R-MAT(a,b,c,d) with 2^scale ids (optionally folded to n nodes), ids permuted by a seeded
    shuffle, self-loops and duplicates removed, 1/in-degree LT weights, suspect_frac random
    suspects with p ~ U(0,1)."""
    nn = 1 << scale
    n = nn if n is None else n
    target = int(edge_factor * n)
    rng = np.random.Generator(np.random.PCG64(seed))
    a, b, c, _ = abcd
    u = np.zeros(target, dtype=np.uint64)
    v = np.zeros(target, dtype=np.uint64)
    for _bit in range(scale):
        r = rng.random(target)
        ubit = r >= a + b
        vbit = ((r >= a) & (r < a + b)) | (r >= a + b + c)
        u = (u << np.uint64(1)) | ubit.astype(np.uint64)
        v = (v << np.uint64(1)) | vbit.astype(np.uint64)
    perm = rng.permutation(nn).astype(np.uint64)
    u, v = perm[u], perm[v]
    if n != nn:
        u, v = u % np.uint64(n), v % np.uint64(n)
    off, src = csr_from_edges(n, u, v)
    cum = indegree_cum(off)
    p_of = random_suspects(n, max(1, int(suspect_frac * n)), suspect_seed)
    return CsrGraph(n, int(off[-1]), off, src, cum, p_of)


def uniform_graph(n: int, density: int, seed: int = 1, suspect_count: int = 10,
                  suspect_seed: int = 2) -> CsrGraph:
    """G(n, n*density) without loops/duplicates (the shape of synth_graph), 1/in-degree weights."""
    rng = np.random.Generator(np.random.PCG64(seed))
    want = n * density
    u = rng.integers(0, n, size=int(want * 1.05) + 16, dtype=np.uint64)
    v = rng.integers(0, n, size=u.size, dtype=np.uint64)
    off, src = csr_from_edges(n, u, v)
    cum = indegree_cum(off)
    p_of = random_suspects(n, suspect_count, suspect_seed)
    return CsrGraph(n, int(off[-1]), off, src, cum, p_of)

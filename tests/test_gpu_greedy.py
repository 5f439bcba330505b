"""GPU parity tests for greedy max-cover and coverage_of (kernels K3-K6), through the C-ABI, in
fixed-walk-set mode: the same item sets go to the device and to the oracle, and the selected items
and coverage must be bit-exact. Mirrors proj/tests/test_coverage.cpp."""
import numpy as np
import pytest

from conftest import make_csr, upload

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["full-ids", "dense"])
def instance_form(request, monkeypatch):
    """Every test of this module runs twice: on the id space as given, and with the dense reduced
    instance forced (greedy.cu build_dense: indexed items renamed 0..D-1, walks restricted to them;
    production uses it from 256 MB of counters upwards, i.e. the LiveJournal shape and beyond)."""
    if request.param == "dense":
        monkeypatch.setenv("HSAW_DENSE_MIN_BYTES", "0")
        monkeypatch.setenv("HSAW_COVERAGE_FLAT", "2")  # and the flat coverage_of kernel
    else:
        monkeypatch.setenv("HSAW_DENSE_MIN_BYTES", str(1 << 60))
        monkeypatch.setenv("HSAW_COVERAGE_FLAT", "0")
    return request.param


def to_csr_sets(sets):
    off = np.zeros(len(sets) + 1, dtype=np.uint64)
    np.cumsum([len(s) for s in sets], out=off[1:])
    items = np.array([x for s in sets for x in s], dtype=np.uint32)
    return off, items


def test_micro_instance(ctx, gpu_lib):  # proj/tests/test_coverage.cpp:43-70
    off, items = to_csr_sets([[1, 2], [2], [3]])
    with ctx.walkset(20, off, items) as ws:
        sol, cov = ctx.greedy(1, walkset=ws)
        assert sol.tolist() == [2] and cov == 2
        sol, cov = ctx.greedy(2, walkset=ws)
        assert sol.tolist() == [2, 3] and cov == 3
        sol, cov = ctx.greedy(3, walkset=ws, cand=[1, 2, 3])
        assert sol.tolist() == [2, 3, 1] and cov == 3  # zero-gain slot padded by smallest id
        with pytest.raises(gpu_lib.HsawError) as e:
            ctx.greedy(4, walkset=ws, cand=[1, 2, 3])
        assert e.value.status == gpu_lib.HSAW_EINVAL
        with pytest.raises(gpu_lib.HsawError) as e:
            ctx.greedy(1, walkset=ws, cand=[1, 2, 20])
        assert e.value.status == gpu_lib.HSAW_EDATA
        # all-zero-gain: every slot is padding, ascending ids (test_interdiction.cpp:66-82)
        sol, cov = ctx.greedy(3, walkset=ws, cand=[7, 5, 9, 11])
        assert sol.tolist() == [5, 7, 9] and cov == 0
        assert ctx.coverage_of([2], walkset=ws) == 2
        assert ctx.coverage_of([1, 3], walkset=ws) == 2
        assert ctx.coverage_of([1, 2, 3], walkset=ws) == 3
        assert ctx.coverage_of([2], walkset=ws, cand=[1, 3]) == 0  # non-candidates are not indexed


def test_golden_instances(ctx, golden):
    for g in golden["greedy"]:
        with ctx.walkset(g["limit"], g["set_off"], g["items"]) as ws:
            sol, cov = ctx.greedy(g["k"], walkset=ws, cand=g["cand"])
            assert sol.tolist() == g["solution"] and cov == g["coverage"]
            assert ctx.coverage_of(g["solution"], walkset=ws, cand=g["cand"]) == g["coverage_of"]


def test_random_instances_match_oracle(ctx, port):
    """test_coverage.cpp:72-93 at larger sizes; sets may repeat an item (multiplicity counts in
    the gain exactly as by_item_ holds the sample twice, coverage.cpp:31-35)."""
    rng = np.random.Generator(np.random.PCG64(7))
    for inst in range(30):
        limit = int(rng.integers(5, 400))
        nsets = int(rng.integers(1, 3000))
        sizes = rng.integers(0, 9, size=nsets)
        zipf = np.minimum(rng.zipf(1.3, size=int(sizes.sum())) - 1, limit - 1)
        items = ((zipf * 7919 + inst) % limit).astype(np.uint32)
        off = np.zeros(nsets + 1, dtype=np.uint64)
        np.cumsum(sizes, out=off[1:])
        cand = None
        if inst % 3 == 1:
            cand = np.unique(rng.integers(0, limit, size=max(2, limit // 3))).astype(np.uint32)
        ncand = limit if cand is None else len(cand)
        k = int(min(1 + inst * 3, ncand))
        exp_sol, exp_cov = port.greedy(limit, off, items, k, cand=cand)
        with ctx.walkset(limit, off, items) as ws:
            sol, cov = ctx.greedy(k, walkset=ws, cand=cand)
            assert sol.tolist() == exp_sol.tolist(), inst
            assert cov == exp_cov
            assert ctx.coverage_of(sol, walkset=ws, cand=cand) == \
                port.coverage_of(limit, off, items, sol, cand=cand)
            sub = (nsets // 3, nsets // 2)
            e2, c2 = port.greedy(limit, off[sub[0]:sub[0] + sub[1] + 1] - off[sub[0]],
                                 items[int(off[sub[0]]):int(off[sub[0] + sub[1]])], min(k, 3),
                                 cand=cand)
            s2, cv2 = ctx.greedy(min(k, 3), walkset=ws, cand=cand, off=sub[0], cnt=sub[1])
            assert s2.tolist() == e2.tolist() and cv2 == c2  # sub-range of the walk set


def test_empty_inputs(ctx):
    off, items = to_csr_sets([[], [], []])
    with ctx.walkset(10, off, items) as ws:
        sol, cov = ctx.greedy(4, walkset=ws)
        assert sol.tolist() == [0, 1, 2, 3] and cov == 0
        assert ctx.coverage_of([1, 2], walkset=ws) == 0
        sol, cov = ctx.greedy(2, walkset=ws, off=1, cnt=0)
        assert sol.tolist() == [0, 1] and cov == 0


@pytest.mark.parametrize("kind", [0, 1])
def test_stream_greedy_matches_oracle(ctx, port, synth3000, kind):
    """Greedy straight on the device-resident stream (edge ids for eSIA, all nodes incl. start
    and hit for nSIA, coverage.cpp:49-53) vs the oracle on the exported walks."""
    upload(ctx, synth3000)
    limit = synth3000.m if kind == 0 else synth3000.n
    with ctx.stream(seed=3) as st:
        st.ensure(6000)
        pool = st.export(0, 6000)
        from oracle.oracle import PoolData
        pd = PoolData(0, pool.edge_off, pool.nodes, pool.edges, pool.tag_worker, pool.tag_seq)
        for off, cnt, k in ((0, 3000, 20), (3000, 3000, 5), (100, 1, 2)):
            so, it = pd.item_sets(kind, off, cnt)
            exp_sol, exp_cov = port.greedy(limit, so, it, k)
            sol, cov = ctx.greedy(k, stream=st, kind=kind, off=off, cnt=cnt)
            assert sol.tolist() == exp_sol.tolist() and cov == exp_cov
            assert ctx.coverage_of(sol, stream=st, kind=kind, off=off, cnt=cnt) == \
                port.coverage_of(limit, so, it, sol)
        cand = np.arange(0, limit, 3, dtype=np.uint32)
        so, it = pd.item_sets(kind, 0, 6000)
        exp_sol, exp_cov = port.greedy(limit, so, it, 15, cand=cand)
        sol, cov = ctx.greedy(15, stream=st, kind=kind, off=0, cnt=6000, cand=cand)
        assert sol.tolist() == exp_sol.tolist() and cov == exp_cov


def test_greedy_is_monotone_submodular(ctx, synth3000):  # test_coverage.cpp:95-124
    upload(ctx, synth3000)
    rng = np.random.Generator(np.random.PCG64(11))
    with ctx.stream(seed=6) as st:
        st.ensure(2000)
        for _ in range(40):
            big = np.unique(rng.integers(0, synth3000.n, size=6)).astype(np.uint32)
            small = big[: len(big) // 2]
            x = int(rng.integers(0, synth3000.n))
            while x in big:
                x = int(rng.integers(0, synth3000.n))
            cov = lambda items: ctx.coverage_of(items, stream=st, kind=1, off=0, cnt=2000)
            cs, cb = cov(small), cov(big)
            assert cs <= cb
            assert cov(np.append(small, x)) - cs >= cov(np.append(big, x)) - cb


def test_thresholded_index_falls_back_to_full(ctx, port):
    """Large flat instance: the inverted index is first built only for high-count items; with k
    large enough the winners drop below that threshold and the run must restart with the full
    index — selections still bit-exact with the oracle."""
    rng = np.random.Generator(np.random.PCG64(3))
    limit, nsets = 60_000, 1_300_000
    items = rng.integers(0, limit, size=nsets).astype(np.uint32)
    off = np.arange(nsets + 1, dtype=np.uint64)
    k = 12_000
    exp_sol, exp_cov = port.greedy(limit, off, items, k)
    with ctx.walkset(limit, off, items) as ws:
        sol, cov = ctx.greedy(k, walkset=ws)
    assert cov == exp_cov and sol.tolist() == exp_sol.tolist()
    # and a skewed one where the threshold holds (no fallback needed)
    z = np.minimum(rng.zipf(1.2, size=nsets * 2) - 1, limit - 1).astype(np.uint32)
    off2 = np.arange(0, 2 * nsets + 1, 2, dtype=np.uint64)
    exp_sol, exp_cov = port.greedy(limit, off2, z, 40)
    with ctx.walkset(limit, off2, z) as ws:
        sol, cov = ctx.greedy(40, walkset=ws)
    assert cov == exp_cov and sol.tolist() == exp_sol.tolist()


def test_flat_counts_above_the_mass_rule(ctx, port):
    """Every item occurs equally often: the 1/8-mass rule lands one above the only count there is,
    so nothing is indexed at the first threshold (an empty dense instance / an unindexed first
    winner) and the run must step down to the full index."""
    limit, reps = 300_000, 4
    items = np.tile(np.arange(limit, dtype=np.uint32), reps)  # > 2^20 occurrences, all counts = 4
    off = np.arange(0, items.size + 1, 3, dtype=np.uint64)
    if off[-1] != items.size:
        off = np.append(off, np.uint64(items.size))
    exp_sol, exp_cov = port.greedy(limit, off, items, 50)
    with ctx.walkset(limit, off, items) as ws:
        sol, cov = ctx.greedy(50, walkset=ws)
    assert cov == exp_cov and sol.tolist() == exp_sol.tolist()


def test_partitioned_histogram_large_id_space(ctx, port):
    """Id spaces whose counters do not fit L2 take the radix-partitioned histogram path."""
    rng = np.random.Generator(np.random.PCG64(9))
    limit, nsets = 13_500_000, 2_400_000
    z = ((np.minimum(rng.zipf(1.15, size=nsets * 2), 10**7) * 2654435761) % limit).astype(np.uint32)
    off = np.arange(0, 2 * nsets + 1, 2, dtype=np.uint64)
    exp_sol, exp_cov = port.greedy(limit, off, z, 25)
    with ctx.walkset(limit, off, z) as ws:
        sol, cov = ctx.greedy(25, walkset=ws)
        assert cov == exp_cov and sol.tolist() == exp_sol.tolist()
        assert ctx.coverage_of(sol, walkset=ws) == port.coverage_of(limit, off, z, sol)


@pytest.mark.parametrize("kind", [0, 1])
def test_coverage_upper_bound(ctx, port, synth3000, kind):
    """hsaw_gpu_coverage_upper_bound: the sum of the k largest per-item occurrence counts (capped at
    the number of walks) — never below what any k candidates, greedy's included, can cover."""
    upload(ctx, synth3000)
    with ctx.stream(seed=11) as st:
        st.ensure(4000)
        pool = st.to_pool(4000)
        nw = 3000
        so, it = port.stream_samples(synth3000, 4000, seed=11).item_sets(kind)
        items = it[: int(so[nw])]
        limit = synth3000.m if kind == 0 else synth3000.n
        counts = np.bincount(items, minlength=limit)
        for k in (1, 5, 40):
            ub = ctx.coverage_upper_bound(k, stream=st, kind=kind, off=0, cnt=nw)
            assert ub == min(int(np.sort(counts)[::-1][:k].sum()), nw)
            sol, cov = ctx.greedy(k, stream=st, kind=kind, off=0, cnt=nw)
            assert cov <= ub
            assert ctx.coverage_of(sol, stream=st, kind=kind, off=0, cnt=nw) <= ub
        cand = np.arange(0, limit, 7, dtype=np.uint32)
        ub = ctx.coverage_upper_bound(3, stream=st, kind=kind, off=0, cnt=nw, cand=cand)
        assert ub == min(int(np.sort(counts[cand])[::-1][:3].sum()), nw)
        assert pool.nsamples >= nw


@pytest.mark.parametrize("shift", [13, 16])
def test_large_maxima_blocks(gpu_lib, monkeypatch, port, shift):
    """Id spaces past ~50 M items (1.47 G edge ids at the Twitter shape) use 2^shift-item maxima
    blocks so that the single-CTA tail kernel still holds every bound in shared memory; forced here
    on instances small enough for the oracle: same selections, gains and padding."""
    monkeypatch.setenv("HSAW_GREEDY_BLOCK_SHIFT", str(shift))
    rng = np.random.Generator(np.random.PCG64(21))
    with gpu_lib.Context(0) as ctx:
        for limit, nsets, k in ((300_000, 200_000, 300), (70_000, 400_000, 2_000), (5, 40, 5)):
            z = ((np.minimum(rng.zipf(1.25, size=nsets * 3), 10**6) * 2654435761) % limit)
            z = z.astype(np.uint32)
            off = np.arange(0, 3 * nsets + 1, 3, dtype=np.uint64)
            exp_sol, exp_cov = port.greedy(limit, off, z, k)
            with ctx.walkset(limit, off, z) as ws:
                sol, cov = ctx.greedy(k, walkset=ws)
                assert cov == exp_cov and sol.tolist() == exp_sol.tolist()

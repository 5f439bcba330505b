"""The device R-MAT generator (csrc/rmat.cu, bench input tooling of SURVEY.md §8d) against the
sequential host generator hsaw::rmat_graph_n: bit-identical ProbGraph arrays for power-of-two and
arbitrary node counts, degenerate sizes, and the same sample stream whether the graph was generated
on the device and installed where it lies or generated on the host and uploaded."""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert (a.n, a.m) == (b.n, b.m)
    for x, y in zip(a.arrays(), b.arrays()):
        assert x.tobytes() == y.tobytes()


@pytest.mark.parametrize("n,raw,seed", [
    (1 << 14, 16 << 14, 1),      # power of two: the rmat_graph(scale, factor) family
    (1 << 16, 16 << 16, 1),
    (50_000, 700_000, 3),        # endpoints >= n are dropped
    (41_653, 1_467_003, 9),      # the Twitter shape scaled by 1e-3: dense enough to deduplicate
    (3, 100, 5), (2, 7, 1), (1000, 0, 1), (1000, 1, 2), (1000, 9, 2),
])
def test_device_generator_equals_host_generator(n, raw, seed):
    from paper_1702_05854_b200 import hostapi
    host = hostapi.Graph.rmat_n(n, raw, seed)
    _same(hostapi.Graph.rmat_device(n, raw, seed), host)
    lean = hostapi.Graph.rmat_device(n, raw, seed, lean=True)
    for x, y in zip(lean.views(), host.views()):
        assert x.tobytes() == y.tobytes()


def test_scale_20_equals_the_c2_bench_graph():
    """BASELINE configs[1]: the graph every C2 number of this repo was measured on."""
    from paper_1702_05854_b200 import hostapi
    host = hostapi.Graph.rmat(20, 16.0, seed=1)
    assert host.m == 16_085_553
    _same(hostapi.Graph.rmat_device(1 << 20, 16 << 20, 1), host)


def _digest(pool):
    h = hashlib.sha256()
    for a in (pool.edge_off, pool.nodes, pool.edges, pool.tag_worker, pool.tag_seq):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("layout", ["compact", "fat"])
def test_installed_where_it_lies_samples_like_the_uploaded_graph(gpu_lib, monkeypatch, layout):
    from paper_1702_05854_b200 import hostapi
    monkeypatch.setenv("HSAW_LAYOUT", layout)
    n, raw = 30_000, 400_000
    p_of = hostapi.random_suspects_n(n, 300, 2)
    host = hostapi.Graph.rmat_n(n, raw, 4)
    assert np.array_equal(p_of, host.random_suspects(300, 2))
    digests = []
    for dg in (hostapi.DeviceGraph.from_rmat(n, raw, 4, p_of),
               hostapi.DeviceGraph.from_rmat(n, raw, 4, p_of, want_host=True),
               hostapi.DeviceGraph(host, p_of)):
        with dg:
            assert (dg.graph.n, dg.graph.m) == (host.n, host.m)
            ctx = gpu_lib.Context.borrow(dg.ctx_handle(), host.n, host.m)
            with ctx.stream(seed=42) as st:
                st.sample_range(0, 4096)
                digests.append(_digest(st.export()))
    assert digests[0] == digests[1] == digests[2]
    # the shell graph is enough for the solver: same result as with the host graph
    with hostapi.DeviceGraph.from_rmat(n, raw, 4, p_of) as dg:
        a = hostapi.interdict(dg.graph, p_of, 0, 5, 0.2, 0.1, seed=42, dg=dg)
    b = hostapi.interdict(host, p_of, 0, 5, 0.2, 0.1, seed=42)
    assert a == b

"""Partitioned sampling on the device: the restricted K1 / K2 kernels and
hsaw::distributed_sample through the host layer against the reference's own outputs
(tests/golden/partition_vectors.npz) and the oracle restatement, on both device layouts.
Mirrors proj/tests/test_partition.cpp:112-197."""
import numpy as np
import pytest

from test_partition_cpu import KEYS, POOL_FIELDS, golden_part, pcsr, pv  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["compact", "fat"])
def pdg(request, monkeypatch, pcsr):  # noqa: F811
    from paper_1702_05854_b200 import hostapi
    monkeypatch.setenv("HSAW_LAYOUT", request.param)
    g = hostapi.Graph.from_csr(pcsr.n, pcsr.m, pcsr.in_offsets, pcsr.in_src, pcsr.in_cum)
    dg = hostapi.DeviceGraph(g, pcsr.p_of)
    yield hostapi, dg
    dg.close()


@pytest.mark.parametrize("key", KEYS)
def test_distributed_sample_matches_reference(pdg, pv, pcsr, key):  # noqa: F811
    hostapi, dg = pdg
    _, _, _, _, _, target, seed = (int(x) for x in pv["params"])
    part = golden_part(pv, key, pcsr.n)
    r = hostapi.distributed_sample(dg, part.assign, np.stack(part.extended), target, seed=seed,
                                   hops=part.hops)
    assert [r["crossings"], r["attempts"]] == pv[f"{key}_scalars"].tolist()
    assert r["targets"] == pv[f"{key}_targets"].tolist()
    assert r["crossing_fraction"] == float(pv[f"{key}_fraction"][0])
    for f in POOL_FIELDS:
        assert np.array_equal(getattr(r["pool"], f), pv[f"{key}_pool_{f}"]), f


def test_uneven_parts_and_zero_quota(pdg, pv, pcsr):  # noqa: F811
    hostapi, dg = pdg
    g = hostapi.Graph.from_csr(pcsr.n, pcsr.m, pcsr.in_offsets, pcsr.in_src, pcsr.in_cum)
    assign, ext = hostapi.partition(g, 4, "hash")  # only to get shapes; the assignment is external
    assign = pv["ext_assign"]
    from oracle.oracle import extend_partition_np, partition_graph_np
    part = extend_partition_np(pcsr, partition_graph_np(pcsr, 4, "external", assign=assign), 1)
    r = hostapi.distributed_sample(dg, part.assign, np.stack(part.extended), 101, seed=11, hops=1)
    assert r["targets"] == pv["ext_targets"].tolist()
    assert [r["crossings"], r["attempts"]] == pv["ext_scalars"].tolist()
    for f in POOL_FIELDS:
        assert np.array_equal(getattr(r["pool"], f), pv[f"ext_pool_{f}"]), f


@pytest.mark.parametrize("window,heuristic", [(0, 0), (3, 0), (2, 2)])
def test_restricted_stream_other_configs(gpu_lib, port, pv, pcsr, window, heuristic):  # noqa: F811
    """The restricted kernels exist for every SamplerConfig the device supports: one part's
    stream against the oracle's orc_part_sample (windows 0 and 3, heuristic None)."""
    part = golden_part(pv, "hash_h1", pcsr.n)
    from oracle.oracle import PART_STRIDE, Partitioning
    one = Partitioning(1, 1, np.zeros(pcsr.n, dtype=np.uint32), [part.base[2]], [part.extended[2]])
    # oracle: a single-part "partitioning" whose base is part 2's nodes gets the whole target
    exp = port.distributed_sample(pcsr, one, 150, seed=3 + 2 * PART_STRIDE, heuristic=heuristic,
                                  window=window)
    with gpu_lib.Context(0) as ctx:
        ctx.upload_graph(pcsr.n, pcsr.m, pcsr.in_offsets, pcsr.in_src, pcsr.in_cum, pcsr.p_of)
        cfg = gpu_lib.SamplerCfg(heuristic, window, 10, 100_000_000)
        with ctx.stream(seed=3 + 2 * PART_STRIDE, cfg=cfg) as st:
            st.restrict(part.base[2], part.extended[2])
            st.ensure(150)
            pool = st.to_pool(150)
            assert st.crossings(150) == exp.crossings and pool.attempts == exp.attempts
            for f in POOL_FIELDS:
                assert np.array_equal(getattr(pool, f), getattr(exp.pool, f)), f
            with pytest.raises(gpu_lib.HsawError):
                st.restrict(part.base[2], part.extended[2])  # too late

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


@pytest.mark.parametrize("window,heuristic", [(0, 0), (3, 0), (2, 2), (2, 1), (0, 1)])
def test_restricted_stream_other_configs(gpu_lib, port, pv, pcsr, window, heuristic):  # noqa: F811
    """The restricted kernels exist for every SamplerConfig the device supports: one part's
    stream against the oracle's orc_part_sample (windows 0 and 3, heuristics None and Floyd)."""
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


def test_cli_partition_and_baseline(pdg, pv, pcsr, tmp_path):  # noqa: F811
    """`hsaw partition --target` and `hsaw baseline` (proj/src/cli.cpp:197-265,292-335) through the
    drop-in CLI: the numbers the library calls give, nlohmann key order."""
    import json
    hostapi, dg = pdg
    g = hostapi.Graph.from_csr(pcsr.n, pcsr.m, pcsr.in_offsets, pcsr.in_src, pcsr.in_cum)
    cache, sus, out = tmp_path / "g.hsaw1", tmp_path / "s.txt", tmp_path / "o.json"
    g.save_cache(cache)
    sus.write_text("".join(f"{v} {float(pcsr.p_of[v])!r}\n" for v in np.nonzero(pcsr.p_of)[0]))
    rc = hostapi.run_cli(["partition", "--graph", str(cache), "--suspects", str(sus), "--parts", "4",
                          "--hops", "1", "--target", "700", "--seed", "7", "--output", str(out)])
    assert rc == 0
    rep = json.loads(out.read_text())
    key = "hash_h1"
    assert [rep["crossings"], rep["attempts"]] == pv[f"{key}_scalars"].tolist()
    assert rep["per_part_targets"] == pv[f"{key}_targets"].tolist() and rep["target"] == 700
    assert rep["accepted"] == pv[f"{key}_pool_edge_off"].size - 1
    assert rep["crossing_fraction"] == float(pv[f"{key}_fraction"][0])
    assert list(rep) == sorted(rep)
    rc = hostapi.run_cli(["baseline", "--graph", str(cache), "--suspects", str(sus), "--method",
                          "infmax-vi", "--mode", "node", "--k", "5", "--seed", "3", "--output",
                          str(out)])
    assert rc == 0
    rep = json.loads(out.read_text())
    s = __import__("oracle.oracle", fromlist=["Port"]).Port().seed_from_worker(3)
    ids, s_after = hostapi.baseline(g, pcsr.p_of, "infmax-vi", 1, 5, s, dg=dg)
    assert rep["ids"] == ids and rep["k"] == 5 and rep["kind"] == "node" and rep["method"] == "infmax-vi"
    est = hostapi.estimate_suspension(g, pcsr.p_of, 1, ids, 0.1, 0.1, s_after, dg=dg)
    assert rep["suspension"] == est["value"] and 0.0 <= rep["ssr"] <= 1.0 and rep["cost"] >= 0.0
    assert list(rep) == sorted(rep)

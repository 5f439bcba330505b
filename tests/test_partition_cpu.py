"""Partitioned sampling, CPU side: the oracle restatement
(oracle/hsaw_oracle.c orc_part_sample + oracle.partition_graph_np / extend_partition_np) and the
host layer's partition_graph / extend_partition (host/partition.cpp) against vectors produced by
the unmodified reference (tests/golden/make_partition_golden.py). Mirrors
proj/tests/test_partition.cpp:112-197."""
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR
from oracle.oracle import Csr, Partitioning, extend_partition_np, part_quotas, partition_graph_np

KEYS = [f"{m}_h{h}" for m in ("hash", "labelprop") for h in (0, 1, 2)]
POOL_FIELDS = ("edge_off", "nodes", "edges", "tag_worker", "tag_seq")


@pytest.fixture(scope="module")
def pv():
    return np.load(os.path.join(GOLDEN_DIR, "partition_vectors.npz"))


@pytest.fixture(scope="module")
def pcsr(pv):
    n = pv["in_offsets"].size - 1
    return Csr(n, pv["in_src"].size, pv["in_offsets"], pv["in_src"], pv["in_cum"], pv["p_of"])


def golden_part(pv, key, n, p=4):
    assign = pv[f"{key}_assign"]
    ext = np.unpackbits(pv[f"{key}_extended"], axis=1)[:, :n]
    base = [np.nonzero(assign == i)[0].astype(np.uint32) for i in range(p)]
    return Partitioning(p, int(key[-1]), assign, base, [ext[i].copy() for i in range(p)])


@pytest.mark.parametrize("key", KEYS)
def test_partition_restatement_matches_reference(pv, pcsr, key):
    method, hops = key.split("_h")
    part = extend_partition_np(pcsr, partition_graph_np(pcsr, 4, method, seed=5), int(hops))
    gold = golden_part(pv, key, pcsr.n)
    assert np.array_equal(part.assign, gold.assign)
    for a, b in zip(part.extended, gold.extended):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("key", KEYS)
def test_distributed_sample_restatement_matches_reference(pv, pcsr, port, key):
    _, _, _, _, _, target, seed = (int(x) for x in pv["params"])
    r = port.distributed_sample(pcsr, golden_part(pv, key, pcsr.n), target, seed=seed)
    assert [r.crossings, r.attempts] == pv[f"{key}_scalars"].tolist()
    assert r.targets == pv[f"{key}_targets"].tolist()
    assert r.crossing_fraction == float(pv[f"{key}_fraction"][0])
    for f in POOL_FIELDS:
        assert np.array_equal(getattr(r.pool, f), pv[f"{key}_pool_{f}"]), f


def test_uneven_parts_and_zero_quota(pv, pcsr, port):
    assign = pv["ext_assign"]
    part = extend_partition_np(pcsr, partition_graph_np(pcsr, 4, "external", assign=assign), 1)
    r = port.distributed_sample(pcsr, part, 101, seed=11)
    assert r.targets == pv["ext_targets"].tolist() == part_quotas(101, [b.size for b in part.base], pcsr.n)
    assert [r.crossings, r.attempts] == pv["ext_scalars"].tolist()
    for f in POOL_FIELDS:
        assert np.array_equal(getattr(r.pool, f), pv[f"ext_pool_{f}"]), f


def test_crossings_shrink_with_hops(pv):  # proj/tests/acceptance.cpp:405-423
    for m in ("hash", "labelprop"):
        cr = [int(pv[f"{m}_h{h}_scalars"][0]) for h in (0, 1, 2)]
        assert cr[0] > cr[1] > cr[2]


@pytest.fixture(scope="module")
def host():
    from paper_1702_05854_b200 import _build, hostapi
    _build.build_all()
    hostapi.lib()
    return hostapi


@pytest.mark.parametrize("key", KEYS)
def test_host_partition_graph_matches_reference(host, pv, pcsr, key, tmp_path):
    """host/partition.cpp: partition_graph (Hash, LabelProp, ExternalFile) + extend_partition."""
    method, hops = key.split("_h")
    g = host.Graph.from_csr(pcsr.n, pcsr.m, pcsr.in_offsets, pcsr.in_src, pcsr.in_cum)
    assign, ext = host.partition(g, 4, method, seed=5, hops=int(hops))
    assert np.array_equal(assign, pv[f"{key}_assign"])
    assert np.array_equal(np.packbits(ext, axis=1), pv[f"{key}_extended"])
    # ExternalFile reads the same assignment back (save_partition's format)
    path = tmp_path / "parts.txt"
    path.write_text("".join(f"{int(a)}\n" for a in assign))
    a2, e2 = host.partition(g, 4, "external", part_file=path, hops=int(hops))
    assert np.array_equal(a2, assign) and np.array_equal(e2, ext)


def test_host_partition_errors(host, pcsr, tmp_path):
    g = host.Graph.from_csr(pcsr.n, pcsr.m, pcsr.in_offsets, pcsr.in_src, pcsr.in_cum)
    for bad_p in (0, pcsr.n + 1):
        with pytest.raises(host.HsawError) as e:
            host.partition(g, bad_p)
        assert "part count must be in [1, n]" in str(e.value)
    short = tmp_path / "short.txt"
    short.write_text("0\n1\n")
    with pytest.raises(host.HsawError) as e:
        host.partition(g, 2, "external", part_file=short)
    assert "part file shorter than n" in str(e.value)
    bad = tmp_path / "bad.txt"
    bad.write_text("5\n" * pcsr.n)
    with pytest.raises(host.HsawError) as e:
        host.partition(g, 2, "external", part_file=bad)
    assert "part id 5 out of range" in str(e.value)


def test_cli_partition_report(host, pv, pcsr, tmp_path):
    """`hsaw partition` without --target needs no device (proj/src/cli.cpp:292-335): part sizes,
    extended sizes and the saved part vector."""
    import json
    g = host.Graph.from_csr(pcsr.n, pcsr.m, pcsr.in_offsets, pcsr.in_src, pcsr.in_cum)
    cache, out, saved = tmp_path / "g.hsaw1", tmp_path / "p.json", tmp_path / "parts.txt"
    g.save_cache(cache)
    rc = host.run_cli(["partition", "--graph", str(cache), "--parts", "4", "--method", "labelprop",
                       "--hops", "1", "--seed", "5", "--save", str(saved), "--output", str(out)])
    assert rc == 0
    rep = json.loads(out.read_text())
    gold = golden_part(pv, "labelprop_h1", pcsr.n)
    assert rep["parts"] == 4 and rep["hops"] == 1 and rep["method"] == "labelprop"
    assert rep["part_sizes"] == [int(b.size) for b in gold.base]
    assert rep["extended_sizes"] == [int(m.sum()) for m in gold.extended]
    assert list(rep) == sorted(rep)  # nlohmann object order
    assert [int(x) for x in saved.read_text().split()] == gold.assign.tolist()
    assert host.run_cli(["partition", "--graph", str(cache), "--parts", "0"]) == 2
    assert host.run_cli(["partition", "--graph", str(cache), "--parts", "2", "--method", "x"]) == 1

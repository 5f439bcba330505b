"""Reverse-reachable node sets and the InfMax baselines on the device:
hsaw_gpu_rr_node_sets against the oracle's sequential restatement (sets and the PrgState after),
and hsaw::baseline against the unmodified reference's outputs. Mirrors
proj/tests/test_evaluation.cpp:201-246."""
import numpy as np
import pytest

from conftest import upload
from oracle.oracle import Csr
from test_baseline_cpu import bv  # noqa: F401
from test_partition_cpu import pcsr, pv  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("count", [0, 1, 7, 3000, 40000])
def test_rr_node_sets_match_oracle(ctx, port, pcsr, count):  # noqa: F811
    upload(ctx, pcsr)
    s0 = port.seed_from_worker(31 + count)
    ws, s1 = ctx.rr_node_sets(s0, count)
    with ws:
        off, items = ws.export()
    eoff, eitems, es = port.rr_node_sets(pcsr, s0, count)
    assert np.array_equal(off, eoff) and np.array_equal(items, eitems) and s1 == es


def test_rr_sets_longer_than_the_speculative_buffer(ctx, port):
    """A directed ring (every node has one in-edge of weight 1): every set walks the whole ring,
    3000 nodes, far past the 1024-node thread-local path of the speculative kernel."""
    n = 3000
    off = np.arange(n + 1, dtype=np.uint64)
    src = ((np.arange(n) + n - 1) % n).astype(np.uint32)
    csr = Csr(n, n, off, src, np.ones(n), np.zeros(n))
    upload(ctx, csr)
    s0 = port.seed_from_worker(5)
    ws, s1 = ctx.rr_node_sets(s0, 9)
    with ws:
        o, items = ws.export()
    eo, ei, es = port.rr_node_sets(csr, s0, 9)
    assert np.array_equal(o, eo) and np.array_equal(items, ei) and s1 == es
    assert np.all(np.diff(o) == n)


def test_rr_sets_feed_the_device_greedy(ctx, port, pcsr):  # noqa: F811
    upload(ctx, pcsr)
    s0 = port.seed_from_worker(77)
    ws, _ = ctx.rr_node_sets(s0, 5000)
    eoff, eitems, _ = port.rr_node_sets(pcsr, s0, 5000)
    with ws:
        sol, cov = ctx.greedy(40, walkset=ws, kind=1)
    esol, ecov = port.greedy(pcsr.n, eoff, eitems, 40, kind=1)
    assert sol.tolist() == esol.tolist() and cov == ecov


@pytest.mark.parametrize("layout", ["compact", "fat"])
def test_infmax_baselines_match_reference(monkeypatch, bv, pcsr, layout):  # noqa: F811
    from paper_1702_05854_b200 import hostapi
    monkeypatch.setenv("HSAW_LAYOUT", layout)
    g = hostapi.Graph.from_csr(pcsr.n, pcsr.m, pcsr.in_offsets, pcsr.in_src, pcsr.in_cum)
    with hostapi.DeviceGraph(g, pcsr.p_of) as dg:
        for c in bv["cases"]:
            if not c["kind"].startswith("infmax"):
                continue
            if "error" in c:
                with pytest.raises(hostapi.HsawError):
                    hostapi.baseline(g, pcsr.p_of, c["kind"], c["mode"], c["k"], bv["state0"],
                                     bv["infmax_samples"], dg=dg)
                continue
            ids, s = hostapi.baseline(g, pcsr.p_of, c["kind"], c["mode"], c["k"], bv["state0"],
                                      bv["infmax_samples"], dg=dg)
            assert ids == c["ids"] and s == c["state"], c
        off, items, s1 = hostapi.rr_node_sets(dg, bv["state0"], 100)
        assert off[-1] == items.size and s1 != bv["state0"]

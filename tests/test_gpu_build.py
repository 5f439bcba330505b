"""GPU parity tests of the device CSR builder (csrc/build.cu) through the C-ABI: bit-exact
in_offsets / in_src / in_cum / weight / edge_dst against the golden vectors of the compiled
reference and the oracle restatement, the reference's error messages, and walks sampled on a graph
built on the device equal to walks on the uploaded reference CSR. Mirrors
proj/tests/test_graph.cpp:24-37,65-93,211-236."""
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR
from oracle.oracle import BuildError, Csr, build_graph_np
from test_build_cpu import BAD, CASES

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bg():
    return np.load(os.path.join(GOLDEN_DIR, "build_graph.npz"))


@pytest.mark.parametrize("name", CASES)
def test_device_build_matches_golden(ctx, bg, name):
    n, mode = int(bg[f"{name}_n"][0]), int(bg[f"{name}_mode"][0])
    w = bg[f"{name}_w"] if mode == 0 else None
    off, src, cum, wt, dst = ctx.build_csr(n, bg[f"{name}_u"], bg[f"{name}_v"], w, mode)
    assert np.array_equal(off, bg[f"{name}_off"]) and np.array_equal(src, bg[f"{name}_src"])
    assert cum.tobytes() == bg[f"{name}_cum"].tobytes()
    assert wt.tobytes() == bg[f"{name}_weight"].tobytes()
    assert np.array_equal(dst, bg[f"{name}_dst"])


def test_device_build_matches_oracle_on_rmat(ctx):
    """A larger instance (staged copies both ways, hub rows): R-MAT edges in shuffled order."""
    from paper_1702_05854_b200 import rmat
    g = rmat.rmat_graph(16, 16, seed=21, suspect_frac=0.01)
    dst = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.in_offsets).astype(np.int64))
    perm = np.random.default_rng(5).permutation(g.m)
    u, v = g.in_src[perm], dst[perm]
    off, src, cum, wt, d2 = ctx.build_csr(g.n, u, v, None, 1)
    assert np.array_equal(off, g.in_offsets) and np.array_equal(src, g.in_src)
    assert cum.tobytes() == np.ascontiguousarray(g.in_cum).tobytes()
    assert np.array_equal(d2, dst)
    eo, es, ec, ew, ed = build_graph_np(g.n, u[:20000], v[:20000], None, 1)
    o2, s2, c2, w2, _ = ctx.build_csr(g.n, u[:20000], v[:20000], None, 1)
    assert np.array_equal(o2, eo) and np.array_equal(s2, es)
    assert c2.tobytes() == ec.tobytes() and w2.tobytes() == ew.tobytes()


@pytest.mark.parametrize("name", list(BAD))
def test_device_build_errors(ctx, gpu_lib, name):
    n, u, v, w, mode, msg = BAD[name]
    with pytest.raises(gpu_lib.HsawError) as e:
        ctx.build_csr(n, np.array(u), np.array(v), None if w is None else np.array(w), mode)
    assert e.value.status == gpu_lib.HSAW_EDATA and msg in str(e.value)


def test_device_build_rejects_hub_rows(ctx, gpu_lib):
    d = 36217
    u = np.arange(1, d + 1, dtype=np.uint32)
    v = np.zeros(d, dtype=np.uint32)
    with pytest.raises(gpu_lib.HsawError) as e:
        ctx.build_csr(d + 1, u, v, None, 1)
    assert "graph: in-weight sum 1.000000 > 1 at node 0" in str(e.value)
    off, _, cum, _, _ = ctx.build_csr(d, u[:-1], v[:-1], None, 1)
    assert int(off[1]) == d - 1 and cum[d - 2] <= 1.0 + 1e-12


def test_random_normalized_is_not_built_on_device(ctx, gpu_lib):
    with pytest.raises(gpu_lib.HsawError) as e:
        ctx.build_csr(3, np.array([0]), np.array([1]), None, 2)
    assert e.value.status == gpu_lib.HSAW_EINVAL


def test_empty_edge_list(ctx):
    off, src, cum, _, _ = ctx.build_csr(4, np.zeros(0, np.uint32), np.zeros(0, np.uint32), None, 1)
    assert off.tolist() == [0] * 5 and src.size == 0 and cum.size == 0


def test_build_upload_samples_like_uploaded_csr(ctx, port, bg):
    """Edge list -> device graph without a host CSR: the pool equals the oracle's stream on the
    reference-built CSR (proj/src/sampler.cpp:388-463)."""
    name = "indeg_hub"
    n = int(bg[f"{name}_n"][0])
    p_of = np.zeros(n)
    rng = np.random.default_rng(3)
    sus = rng.choice(n, size=n // 50, replace=False)
    p_of[sus] = rng.uniform(0.05, 1.0, size=sus.size)
    ctx.build_upload_graph(n, bg[f"{name}_u"], bg[f"{name}_v"], p_of, None, 1)
    with ctx.stream(seed=9) as st:
        st.ensure(2000)
        got = st.to_pool(2000)
    csr = Csr(n, bg[f"{name}_src"].size, bg[f"{name}_off"], bg[f"{name}_src"], bg[f"{name}_cum"],
              p_of)
    exp = port.stream_samples(csr, 2000, seed=9)
    assert got.attempts == exp.attempts and got.nsamples == exp.nsamples
    assert np.array_equal(got.nodes, exp.nodes) and np.array_equal(got.edges, exp.edges)


@pytest.mark.parametrize("name", ["indeg_hub", "given"])
def test_host_layer_build_graph_device(bg, name):
    """hsaw::build_graph_device (host layer, C++): the same ProbGraph as the reference's build_graph
    — every field, bit for bit — and the reference's DataError on bad input."""
    from paper_1702_05854_b200 import hostapi
    n, mode = int(bg[f"{name}_n"][0]), int(bg[f"{name}_mode"][0])
    w = bg[f"{name}_w"] if mode == 0 else None
    g = hostapi.Graph.build_device(n, bg[f"{name}_u"], bg[f"{name}_v"], w, mode)
    off, src, cum, wt, dst = g.arrays()
    assert np.array_equal(off, bg[f"{name}_off"]) and np.array_equal(src, bg[f"{name}_src"])
    assert cum.tobytes() == bg[f"{name}_cum"].tobytes()
    assert wt.tobytes() == bg[f"{name}_weight"].tobytes() and np.array_equal(dst, bg[f"{name}_dst"])
    g.validate()
    with pytest.raises(hostapi.HsawError) as e:
        hostapi.Graph.build_device(3, np.array([0, 2, 0]), np.array([1, 1, 1]))
    assert "duplicate edge 0 -> 1" in str(e.value)

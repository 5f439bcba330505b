"""Binary ingest on the device: HSAW1 cache images written by the reference's
save_cache (proj/src/graph.cpp:383-396) decoded by hsaw_gpu_cache_decode / installed by
hsaw_gpu_graph_cache_upload, against the arrays the reference's load_cache (:398-430) returns for
the same files and the DataError messages it raises for corrupted ones (tests/golden/
cache_vectors.npz, cache_errors.json; generator make_cache_golden.py)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, upload

pytestmark = pytest.mark.gpu

NAMES = ("fixture12", "synth300", "synth2000_random")


@pytest.fixture(scope="module")
def vec():
    return np.load(os.path.join(GOLDEN_DIR, "cache_vectors.npz"))


@pytest.fixture(scope="module")
def errors():
    with open(os.path.join(GOLDEN_DIR, "cache_errors.json")) as f:
        return json.load(f)


def _same(got, vec, name):
    off, src, cum, w, dst = got
    assert np.array_equal(off, vec[name + "_off"])
    assert np.array_equal(src, vec[name + "_src"])
    assert np.array_equal(cum.view(np.uint64), vec[name + "_cum"].view(np.uint64))  # bit-exact
    assert np.array_equal(w.view(np.uint64), vec[name + "_weight"].view(np.uint64))
    assert np.array_equal(dst, vec[name + "_dst"])


def test_decode_matches_reference_load_cache(gpu_lib, vec):
    with gpu_lib.Context(0) as ctx:
        for name in NAMES:
            _same(ctx.decode_cache(vec[name + "_image"].tobytes()), vec, name)


def test_host_layer_load_cache_device(vec, tmp_path):
    from paper_1702_05854_b200 import hostapi
    for name in NAMES:
        path = tmp_path / (name + ".hsaw1")
        path.write_bytes(vec[name + "_image"].tobytes())
        g = hostapi.Graph.load_cache_device(path)
        _same(g.arrays(), vec, name)
        h = hostapi.Graph.load_cache(path)  # the host loader, same file
        for a, b in zip(g.arrays(), h.arrays()):
            assert np.array_equal(a, b)


def test_corrupted_images_raise_the_reference_messages(vec, errors, tmp_path):
    from paper_1702_05854_b200 import hostapi
    for name, want in errors.items():
        path = tmp_path / (name + ".hsaw1")
        path.write_bytes(vec["bad_" + name].tobytes())
        with pytest.raises(hostapi.HsawError) as ei:
            hostapi.Graph.load_cache_device(path)
        assert ei.value.status == 2, name
        assert want.replace("<path>", str(path)) in str(ei.value), (name, str(ei.value))
        with pytest.raises(hostapi.HsawError) as ei:
            hostapi.DeviceGraph.from_cache(path)
        assert ei.value.status == 2, name
        assert want.replace("<path>", str(path)) in str(ei.value), (name, str(ei.value))
    with pytest.raises(hostapi.HsawError) as ei:
        hostapi.Graph.load_cache_device(tmp_path / "missing.hsaw1")
    assert ei.value.status == 2 and "cannot open cache" in str(ei.value)


def test_cache_upload_samples_like_csr_upload(ctx, gpu_lib, vec):
    """file -> resident graph (no host CSR) gives the same walk stream as uploading the arrays."""
    rng = np.random.Generator(np.random.PCG64(4))
    for name in ("synth300", "synth2000_random"):
        off, src, cum = vec[name + "_off"], vec[name + "_src"], vec[name + "_cum"]
        n, m = off.size - 1, src.size
        p_of = np.zeros(n)
        p_of[rng.choice(n, 12, replace=False)] = rng.uniform(0.1, 1.0, 12)
        ctx.upload_graph(n, m, off, src, cum, p_of)
        a = ctx.encode_batches(100, 300)
        ctx.upload_cache(vec[name + "_image"].tobytes(), p_of)
        b = ctx.encode_batches(100, 300)
        for x, y in zip(a[:3], b[:3]):
            assert np.array_equal(x, y), name


def test_from_cache_then_set_suspects(vec, tmp_path):
    from paper_1702_05854_b200 import hostapi
    name = "synth2000_random"
    path = tmp_path / "g.hsaw1"
    path.write_bytes(vec[name + "_image"].tobytes())
    g = hostapi.Graph.load_cache(path)
    p_of = g.random_suspects(20, seed=3)
    with hostapi.DeviceGraph(g, p_of) as dg:
        want = dg.sample(500, seed=9)
        est = hostapi.estimate_suspension(g, p_of, 1, [1, 2, 3], 0.3, 0.2, 5, dg=dg)
    with hostapi.DeviceGraph.from_cache(path) as dg:
        dg.set_suspects(g, p_of)
        assert dg.sample(500, seed=9) == want
        assert hostapi.estimate_suspension(g, p_of, 1, [1, 2, 3], 0.3, 0.2, 5, dg=dg) == est


def test_full_size_cache_round_trip(tmp_path):
    """C2 shape: 386 MB cache file; device ingest equals the host loader on every array."""
    from paper_1702_05854_b200 import hostapi
    g = hostapi.Graph.rmat(20, 16.0, seed=1)
    path = tmp_path / "c2.hsaw1"
    g.save_cache(path)
    # R-MAT hub rows can exceed validate()'s 1e-12 sum tolerance: whatever the host
    # loader does with this file — accept it or reject it — the device loader must do the same
    def load(fn):
        try:
            return fn(path), None
        except hostapi.HsawError as e:
            return None, (e.status, str(e).split(": ", 1)[1])
    (a, ea), (b, eb) = load(hostapi.Graph.load_cache), load(hostapi.Graph.load_cache_device)
    assert ea == eb
    if a is not None:
        for x, y in zip(a.arrays(), b.arrays()):
            assert np.array_equal(x, y)
        with hostapi.DeviceGraph.from_cache(path) as dg:
            p_of = g.random_suspects(g.n // 100, seed=2)
            dg.set_suspects(g, p_of)
            with hostapi.DeviceGraph(g, p_of) as dg2:
                assert dg.sample(100000, seed=42) == dg2.sample(100000, seed=42)


def test_edgeless_cache(tmp_path):
    """A cache with nodes but no edges (offsets all zero) loads the same way on both paths."""
    import struct
    from paper_1702_05854_b200 import hostapi
    path = tmp_path / "empty.hsaw1"
    path.write_bytes(b"HSAW1" + struct.pack("<QQ", 3, 0) + struct.pack("<4Q", 0, 0, 0, 0))
    a, b = hostapi.Graph.load_cache(path), hostapi.Graph.load_cache_device(path)
    assert (a.n, a.m) == (b.n, b.m) == (3, 0)
    assert np.array_equal(a.arrays()[0], b.arrays()[0])
    with hostapi.DeviceGraph.from_cache(path) as dg:
        dg.set_suspects(a, np.array([0.5, 0.0, 1.0]))
        assert dg.sample(10, seed=1)[1] >= 10

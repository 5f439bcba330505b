"""Shared fixtures. `-m "not gpu"` covers the oracle, the host logic and the C-ABI surface on CPU;
`-m gpu` holds the parity tests proper (CUDA path vs oracle), which call through the C-ABI."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def _hexlist(xs):
    return np.array([float.fromhex(x) for x in xs], dtype=np.float64)


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "reference_vectors.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle
    oracle.build()
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return oracle.Ref()


@pytest.fixture(scope="session")
def fixture12(golden):
    """fixture12 with the given weights and the suspects file (CSR produced by the reference)."""
    from oracle.oracle import Csr
    fx = golden["fixture12_given"]
    return Csr(fx["n"], fx["m"], np.array(fx["in_offsets"], dtype=np.uint64),
               np.array(fx["in_src"], dtype=np.uint32), _hexlist(fx["in_cum"]),
               _hexlist(fx["p_of"]))


@pytest.fixture(scope="session")
def fixture12_indegree(golden, fixture12):
    """BASELINE config 1: fixture12 topology, 1/in-degree weights, 10 random suspects (seed 42)."""
    from oracle.oracle import Csr
    c1 = golden["config1_indegree"]["seed42"]
    return Csr(fixture12.n, fixture12.m, fixture12.in_offsets, fixture12.in_src,
               _hexlist(c1["in_cum"]), _hexlist(c1["p_of"]))


@pytest.fixture(scope="session")
def synth3000():
    from oracle.oracle import Csr
    z = np.load(os.path.join(GOLDEN_DIR, "synth3000.npz"))
    n = z["in_offsets"].size - 1
    return Csr(n, z["in_src"].size, z["in_offsets"], z["in_src"], z["in_cum"], z["p_of"])


def make_csr(g):
    """paper_1702_05854_b200.rmat.CsrGraph -> oracle Csr view (same arrays)."""
    from oracle.oracle import Csr
    return Csr(g.n, g.m, g.in_offsets, g.in_src, g.in_cum, g.p_of)


@pytest.fixture(scope="session")
def gpu_lib():
    from paper_1702_05854_b200 import capi
    return capi


# Device graph layouts, chosen at upload time: the L2-resident compact arrays with
# arithmetic picks, the same with every pick forced through the exact threshold path, and the fat
# 32-byte edge records used when the graph outgrows L2. Every parity test runs on all of them.
LAYOUTS = {
    "compact": {"HSAW_LAYOUT": "compact"},  # bit-packed sources with dead-end flags
    "compact-plain": {"HSAW_LAYOUT": "compact", "HSAW_PACK": "0"},  # plain 32-bit sources
    "compact-exact": {"HSAW_LAYOUT": "compact", "HSAW_FORCE_EXACT": "1"},
    "fat": {"HSAW_LAYOUT": "fat"},
}


@pytest.fixture(params=list(LAYOUTS))
def ctx(request, gpu_lib, monkeypatch):
    """A fresh device context per test and graph layout (the CUDA extension must be present: no
    fallback)."""
    monkeypatch.delenv("HSAW_FORCE_EXACT", raising=False)
    monkeypatch.delenv("HSAW_PACK", raising=False)
    for k, v in LAYOUTS[request.param].items():
        monkeypatch.setenv(k, v)
    c = gpu_lib.Context(0)
    yield c
    c.close()


def upload(ctx, csr):
    ctx.upload_graph(csr.n, csr.m, csr.in_offsets, csr.in_src, csr.in_cum, csr.p_of)
    return ctx

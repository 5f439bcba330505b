"""CPU checks of the build_graph restatement (oracle.build_graph_np) against the golden vectors
generated with the compiled reference (tests/golden/make_build_golden.py) and, where oracle/_ref
is present, against the reference live — including its error messages
(proj/src/graph.cpp:112-199, validate :70-104; proj/tests/test_graph.cpp:24-37,65-93)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR
from oracle import oracle
from oracle.oracle import BuildError, build_graph_np

CASES = ["indeg_small", "indeg_hub", "given"]


@pytest.fixture(scope="module")
def bg():
    return np.load(os.path.join(GOLDEN_DIR, "build_graph.npz"))


@pytest.mark.parametrize("name", CASES)
def test_restatement_matches_golden(bg, name):
    n, mode = int(bg[f"{name}_n"][0]), int(bg[f"{name}_mode"][0])
    w = bg[f"{name}_w"] if mode == 0 else None
    off, src, cum, wt, dst = build_graph_np(n, bg[f"{name}_u"], bg[f"{name}_v"], w, mode)
    assert np.array_equal(off, bg[f"{name}_off"]) and np.array_equal(src, bg[f"{name}_src"])
    assert cum.tobytes() == bg[f"{name}_cum"].tobytes()  # bit-exact doubles
    assert wt.tobytes() == bg[f"{name}_weight"].tobytes()
    assert np.array_equal(dst, bg[f"{name}_dst"])


def test_indegree_grid_matches_reference_test():
    """proj/tests/test_graph.cpp:24-37: cumulative grid k/d of a 4-in-edge row."""
    u = np.array([1, 2, 3, 4], dtype=np.uint32)
    v = np.zeros(4, dtype=np.uint32)
    _, _, cum, wt, _ = build_graph_np(5, u, v, None, 1)
    assert cum.tolist() == [0.25, 0.5, 0.75, 1.0] and wt.tolist() == [0.25] * 4


BAD = {
    "range": (3, [0, 5], [1, 2], None, 1, "edge endpoint out of range"),
    "loop": (3, [0, 2], [1, 2], None, 1, "self-loop 2 -> 2"),
    "dup": (3, [0, 2, 0], [1, 1, 1], None, 1, "duplicate edge 0 -> 1"),
    "weight": (3, [0, 2], [1, 1], [0.5, 1.5], 0, "weight 1.500000 out of (0,1] on edge 2 -> 1"),
    "sum": (3, [0, 2], [1, 1], [0.75, 0.5], 0, "in-weight sum 1.250000 > 1 at node 1"),
}


@pytest.mark.parametrize("name", list(BAD))
def test_error_messages(name):
    n, u, v, w, mode, msg = BAD[name]
    with pytest.raises(BuildError) as e:
        build_graph_np(n, u, v, w, mode)
    assert str(e.value) == msg
    if oracle.have_ref():  # the reference says the same
        with pytest.raises(oracle.OracleError) as r:
            oracle.Ref().build_graph(n, np.array(u), np.array(v), None if w is None else np.array(w),
                                     mode=mode)
        assert msg in str(r.value)


def test_hub_row_rejected_like_the_reference():
    """validate() rejects 1/d rows from d = 36 217 on (row sum > 1 + 1e-12)."""
    d = 36217
    u = np.arange(1, d + 1, dtype=np.uint32)
    v = np.zeros(d, dtype=np.uint32)
    with pytest.raises(BuildError) as e:
        build_graph_np(d + 1, u, v, None, 1)
    assert str(e.value) == "graph: in-weight sum 1.000000 > 1 at node 0"
    build_graph_np(d, u[:-1], v[:-1], None, 1)  # 36 216 passes

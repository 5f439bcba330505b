"""CPU suite for the C++ host layer (paper_1702_05854_b200/host): loaders, builders, cache format,
generators, schedule and stopping rule — the host logic either side of the device path. Compared
with committed reference outputs and, where oracle/_ref is built, with the reference itself
(bit-exact arrays). Mirrors proj/tests/test_graph.cpp and test_coverage.cpp:162-242."""
import math
import os

import numpy as np
import pytest

from conftest import _hexlist


@pytest.fixture(scope="module")
def host():
    from paper_1702_05854_b200 import _build, hostapi
    _build.build_all()
    hostapi.lib()
    return hostapi


def same_graph(a, b_arrays):
    off, src, cum, w, dst = a.arrays()
    roff, rsrc, rcum, rw, rdst = b_arrays
    assert np.array_equal(off, roff) and np.array_equal(src, rsrc) and np.array_equal(dst, rdst)
    assert np.array_equal(cum.view(np.uint64), np.asarray(rcum).view(np.uint64))
    assert np.array_equal(w.view(np.uint64), np.asarray(rw).view(np.uint64))


def ref_arrays(ref, gh):
    c = ref._to_csr(gh)
    w, d = ref.graph_extra(gh)
    return c.in_offsets, c.in_src, c.in_cum, w, d


def write_fixture12(path, golden, with_weights=True):
    fx = golden["fixture12_given"]
    w = _hexlist(fx["weight"])
    with open(path, "w") as f:
        f.write("# 12-node demo network\n\n")
        for e in range(fx["m"]):
            if with_weights:
                f.write(f"{fx['in_src'][e]} {fx['edge_dst'][e]} {float(w[e])!r}\n")
            else:
                f.write(f"  {fx['in_src'][e]}\t{fx['edge_dst'][e]}\n")


def test_load_edge_list_fixture12(host, golden, fixture12, tmp_path):
    path = tmp_path / "fixture12.edges"
    write_fixture12(path, golden)
    g = host.Graph.load_edge_list(path, host.WEIGHT_GIVEN)
    off, src, cum, w, dst = g.arrays()
    assert (g.n, g.m) == (12, 20)
    assert np.array_equal(off, fixture12.in_offsets) and np.array_equal(src, fixture12.in_src)
    assert np.array_equal(cum.view(np.uint64), fixture12.in_cum.view(np.uint64))
    assert not os.path.exists(str(path) + ".nodemap")  # ids already dense
    # suspects file: "node prob" per line
    sp = tmp_path / "fixture12.suspects"
    sp.write_text("2 1.0\n5 0.8\n# comment\n9 0.6\n")
    assert np.array_equal(g.load_suspects(sp), fixture12.p_of)


def test_indegree_grid_and_cum(host, golden, tmp_path):
    """proj/tests/test_graph.cpp:24-37: 1/d_in weights, sequential cumulative sums."""
    path = tmp_path / "f.edges"
    write_fixture12(path, golden, with_weights=False)
    g = host.Graph.load_edge_list(path, host.WEIGHT_INDEGREE)
    off, src, cum, w, dst = g.arrays()
    c1 = _hexlist(golden["config1_indegree"]["seed42"]["in_cum"])
    assert np.array_equal(cum.view(np.uint64), c1.view(np.uint64))
    for v in range(g.n):
        d = int(off[v + 1] - off[v])
        s = 0.0
        for e in range(int(off[v]), int(off[v + 1])):
            assert w[e] == 1.0 / d
            s += 1.0 / d
            assert cum[e] == s
    assert np.array_equal(g.random_suspects(10, 42).view(np.uint64),
                          _hexlist(golden["config1_indegree"]["seed42"]["p_of"]).view(np.uint64))


def test_loader_error_paths(host, tmp_path):  # proj/tests/test_graph.cpp:65-93
    def load(text, mode=host.WEIGHT_INDEGREE):
        p = tmp_path / "bad.edges"
        p.write_text(text)
        return host.Graph.load_edge_list(p, mode)

    for text in ("0 1\n1 x\n", "0 1 0.5 extra\n", "0\n", "0 1 0.5x\n", "# only comments\n",
                 "0 0\n", "0 1\n0 1\n", "1.5 2\n"):
        with pytest.raises(host.HsawError) as e:
            load(text)
        assert e.value.status == 2, text
    with pytest.raises(host.HsawError) as e:
        load("0 1\n", host.WEIGHT_GIVEN)  # weight required
    assert e.value.status == 2
    for text in ("0 1 0\n", "0 1 1.5\n", "0 2 0.7\n1 2 0.6\n"):  # weight range, row sum > 1
        with pytest.raises(host.HsawError) as e:
            load(text, host.WEIGHT_GIVEN)
        assert e.value.status == 2
    with pytest.raises(host.HsawError) as e:
        host.Graph.load_edge_list(tmp_path / "missing.edges")
    assert e.value.status == 2


def test_id_remap_and_nodemap(host, tmp_path):  # proj/tests/test_graph.cpp:95-110
    p = tmp_path / "sparse.edges"
    p.write_text("100 7\n7 5000000000\n5000000000 100\n")
    g = host.Graph.load_edge_list(p)
    assert (g.n, g.m) == (3, 3)
    assert (tmp_path / "sparse.edges.nodemap").read_text() == "7 0\n100 1\n5000000000 2\n"
    off, src, *_ = g.arrays()
    assert off.tolist() == [0, 1, 2, 3] and src.tolist() == [1, 2, 0]
    g2 = host.Graph.load_edge_list(p, symmetrize=True, mapping_out=str(tmp_path / "m.txt"))
    assert g2.m == 6 and (tmp_path / "m.txt").exists()


def test_validate_rejects_hub_rows(host):
    """validate() rejects 1/d rows from d = 36217 (drift > 1e-12); 36216 passes."""
    for d, ok in ((36216, True), (36217, False)):
        u = np.arange(1, d + 1, dtype=np.uint32)
        v = np.zeros(d, dtype=np.uint32)
        if ok:
            assert host.Graph.build(d + 1, u, v).m == d
        else:
            with pytest.raises(host.HsawError) as e:
                host.Graph.build(d + 1, u, v)
            assert e.value.status == 2


def test_cache_and_edge_list_round_trip(host, tmp_path):  # test_graph.cpp:211-236
    g = host.Graph.synth(500, 6, 9)
    g.save_cache(tmp_path / "g.cache")
    assert (tmp_path / "g.cache").read_bytes()[:5] == b"HSAW1"
    same_graph(host.Graph.load_cache(tmp_path / "g.cache"), g.arrays())
    g.save_edge_list(tmp_path / "g.edges")
    same_graph(host.Graph.load_edge_list(tmp_path / "g.edges", host.WEIGHT_GIVEN), g.arrays())
    (tmp_path / "bad.cache").write_bytes(b"HSAW2" + b"\0" * 64)
    with pytest.raises(host.HsawError) as e:
        host.Graph.load_cache(tmp_path / "bad.cache")
    assert e.value.status == 2
    blob = (tmp_path / "g.cache").read_bytes()
    (tmp_path / "cut.cache").write_bytes(blob[: len(blob) // 2])
    with pytest.raises(host.HsawError) as e:
        host.Graph.load_cache(tmp_path / "cut.cache")
    assert e.value.status == 2


def test_empty_cache_is_accepted_like_the_reference(host, tmp_path):
    """An HSAW1 cache with n = 0, m = 0 passes the reference's load_cache + validate()
    (proj/src/graph.cpp:76-77, 398-430): both loaders return the empty graph; a non-zero single
    offset or m > 0 is the reference's coverage error. Needs no device."""
    import struct
    (tmp_path / "empty.cache").write_bytes(b"HSAW1" + struct.pack("<QQQ", 0, 0, 0))
    for loader in (host.Graph.load_cache, host.Graph.load_cache_device):
        g = loader(tmp_path / "empty.cache")
        assert (g.n, g.m) == (0, 0)
    (tmp_path / "off.cache").write_bytes(b"HSAW1" + struct.pack("<QQQ", 0, 0, 7))
    for loader in (host.Graph.load_cache, host.Graph.load_cache_device):
        with pytest.raises(host.HsawError) as e:
            loader(tmp_path / "off.cache")
        assert e.value.status == 2 and "offsets do not cover edge range" in str(e.value)


def test_schedule_and_check(host, golden):
    s = host.schedule(100, 2, 0.1, 0.1)  # proj/tests/test_coverage.cpp:162-175
    assert (s["t_max"], s["lambda_samples"]) == (10, 1179)
    assert s["n_max"] == pytest.approx(346869.98374736388, rel=1e-12)
    for row in golden["schedule"]:  # bit-exact with the compiled reference
        s = host.schedule(row["M"], row["k"], row["eps"], row["delta"])
        for key in ("n_max", "lambda_", "lambda1", "t_max", "lambda_samples"):
            assert s[key] == row[key], (row, key)
    ok, e = host.check(1179, 1179, 1179, 100, 2, 0.1, 0.1, 1)  # test_coverage.cpp:213-242
    assert not ok and math.isinf(e)
    ok, e = host.check(2358, 2358, 2358, 100, 2, 0.1, 0.1, 2)
    assert ok and e == pytest.approx(0.0731038970623316, rel=1e-12)
    for args in [(10, 1, 0.0, 0.1), (10, 1, 1.0, 0.1), (10, 1, 0.1, 0.0), (10, 1, 0.1, 1.0),
                 (10, 11, 0.1, 0.1), (10, 0, 0.1, 0.1)]:
        with pytest.raises(host.HsawError) as ex:
            host.schedule(*args)
        assert ex.value.status == 1


def test_check_matches_oracle(host, port):
    rng = np.random.Generator(np.random.PCG64(5))
    for _ in range(200):
        M = int(rng.integers(10, 10**7))
        k = int(rng.integers(1, min(M, 50)))
        eps, delta = float(rng.uniform(0.05, 0.5)), float(rng.uniform(0.01, 0.4))
        n_rp = int(rng.integers(100, 10**6))
        cov_rp = int(rng.integers(0, n_rp))
        cov_r = int(rng.integers(0, n_rp))
        t = int(rng.integers(1, 12))
        a = host.check(cov_r, cov_rp, n_rp, M, k, eps, delta, t)
        b = port.check(cov_r, cov_rp, n_rp, M, k, eps, delta, t)
        assert a[0] == b[0] and (a[1] == b[1] or (math.isinf(a[1]) and math.isinf(b[1])))


def test_rmat_generator_properties(host):
    g = host.Graph.rmat(12, 8, seed=1)
    off, src, cum, w, dst = g.arrays()
    assert g.n == 4096 and 0.8 * 8 * 4096 < g.m <= 8 * 4096
    for v in range(0, g.n, 37):  # sorted, loop-free, distinct sources per row; sequential cum
        row = src[int(off[v]):int(off[v + 1])]
        assert np.all(np.diff(row.astype(np.int64)) > 0) and v not in row
        s = 0.0
        for e in range(int(off[v]), int(off[v + 1])):
            s += 1.0 / len(row)
            assert cum[e] == s
    g2 = host.Graph.rmat(12, 8, seed=1)
    assert np.array_equal(g2.arrays()[1], src)  # deterministic
    deg = np.diff(off.astype(np.int64))
    assert deg.max() > 20 * deg.mean()  # heavy-tailed in-degrees


def test_cli_cpu_paths(host, tmp_path, golden):
    """Exit codes of proj/src/cli.cpp:520-538 on the paths that need no device."""
    assert host.run_cli(["interdict", "--graph", "x"]) == 1          # --k required
    assert host.run_cli(["frobnicate"]) == 1
    assert host.run_cli(["interdict", "--graph", "x", "--k", "1", "--bogus", "1"]) == 1
    assert host.run_cli(["interdict", "--graph", str(tmp_path / "nope"), "--k", "1",
                         "--random-suspects", "2"]) == 2              # data error
    assert host.run_cli(["synth", "--nodes", "50", "--density", "3", "--seed", "4", "--out",
                         str(tmp_path / "s.edges"), "--cache", str(tmp_path / "s.cache")]) == 0
    a = host.Graph.load_cache(tmp_path / "s.cache")
    same_graph(host.Graph.synth(50, 3, 4), a.arrays())
    assert host.run_cli(["synth", "--nodes", "1"]) == 2
    import torch
    if not torch.cuda.is_available():
        path = tmp_path / "fixture12.edges"
        write_fixture12(path, golden)
        # no CUDA device: the device path fails loudly (runtime error, exit 3) — no CPU fallback
        assert host.run_cli(["interdict", "--graph", str(path), "--weights", "given", "--k", "3",
                             "--random-suspects", "3"]) == 3


# ---- against the compiled reference (only in the build container) ------------------------------
def test_generators_match_reference(host, ref):
    for n, d, seed in ((300, 5, 21), (2000, 3, 7), (50, 10, 0)):
        gh = ref.synth_graph(n, d, seed)
        g = host.Graph.synth(n, d, seed)
        same_graph(g, ref_arrays(ref, gh))
        for count, s2 in ((30, 4), (n // 3, 99)):
            assert np.array_equal(g.random_suspects(count, s2).view(np.uint64),
                                  ref.random_suspects(gh, count, s2).view(np.uint64))
        ref.graph_free(gh)


def test_build_graph_modes_match_reference(host, ref):
    rng = np.random.Generator(np.random.PCG64(3))
    n = 400
    pairs = set()
    while len(pairs) < 3000:
        u, v = int(rng.integers(0, n)), int(rng.integers(0, n))
        if u != v:
            pairs.add((u, v))
    u = np.array([p[0] for p in pairs], dtype=np.uint32)
    v = np.array([p[1] for p in pairs], dtype=np.uint32)
    w = rng.uniform(0.001, 0.05, size=u.size)
    for mode in (0, 1, 2):
        gh = ref.build_graph(n, u, v, w, mode=mode, seed=17)
        same_graph(host.Graph.build(n, u, v, w, mode=mode, seed=17), ref_arrays(ref, gh))
        ref.graph_free(gh)


def test_file_formats_match_reference(host, ref, tmp_path):
    gh = ref.synth_graph(700, 4, 5)
    g = host.Graph.synth(700, 4, 5)
    ref.save_cache(gh, str(tmp_path / "ref.cache"))
    g.save_cache(tmp_path / "mine.cache")
    assert (tmp_path / "ref.cache").read_bytes() == (tmp_path / "mine.cache").read_bytes()
    ref.save_edge_list(gh, str(tmp_path / "ref.edges"))
    g.save_edge_list(tmp_path / "mine.edges")
    assert (tmp_path / "ref.edges").read_text() == (tmp_path / "mine.edges").read_text()
    same_graph(host.Graph.load_cache(tmp_path / "ref.cache"), ref_arrays(ref, gh))
    (tmp_path / "odd.edges").write_text("# c\n 9 4 \n4 9\n\n17 9\n9 17\n4 17\n")
    for sym in (False, True):
        rh = ref.load_edge_list(str(tmp_path / "odd.edges"), mode=2, seed=3, symmetrize=sym,
                                mapping_out=str(tmp_path / "r.map"))
        mine = host.Graph.load_edge_list(tmp_path / "odd.edges", 2, 3, symmetrize=sym,
                                         mapping_out=str(tmp_path / "m.map"))
        same_graph(mine, ref_arrays(ref, rh))
        assert (tmp_path / "r.map").read_text() == (tmp_path / "m.map").read_text()
        ref.graph_free(rh)
    ref.graph_free(gh)


def test_json_numbers_follow_nlohmann_layout(host):
    """to_json (proj/src/interdiction.cpp:89-104) prints doubles as nlohmann::json::dump does:
    fixed notation while the decimal exponent is in (-4, 15], else d.ddde+-XX. Expected strings
    were produced by nlohmann 3.11.3 itself."""
    cases = {1e-4: "0.0001", 1e5: "100000.0", 1e6: "1000000.0", 0.1: "0.1", 3.0: "3.0",
             2.0664354087995083: "2.0664354087995083", 1e15: "1e+15", 123456789012345.0: "123456789012345.0",
             1e16: "1e+16", 1.5e-5: "1.5e-05", 9.5367431640625e-07: "9.5367431640625e-07",
             1.2345678901234568e+17: "1.2345678901234568e+17", 0.00012345: "0.00012345",
             12345.678: "12345.678", -2.5: "-2.5", -1e-7: "-1e-07", 1e22: "1e+22",
             5e-324: "5e-324", 804.4299041134876: "804.4299041134876", 0.0: "0.0"}
    for x, want in cases.items():
        assert host.json_number(x) == want, x


def test_rmat_n_generalises_rmat(host):
    """rmat_graph(scale, f) is rmat_graph_n(2^scale, floor(f 2^scale)); other node counts drop raw
    edges with an endpoint >= n; suspects depend on the node count only."""
    a, b = host.Graph.rmat(12, 8.0, seed=3), host.Graph.rmat_n(1 << 12, 8 << 12, seed=3)
    assert all(np.array_equal(x, y) for x, y in zip(a.arrays(), b.arrays()))
    g = host.Graph.rmat_n(3000, 40000, seed=3)
    off, src, cum, w, dst = g.arrays()
    assert g.n == 3000 and 0 < g.m < 40000 and src.max() < 3000 and off[-1] == g.m
    key = dst.astype(np.int64) * g.n + src
    assert np.all(np.diff(key) > 0) and not np.any(src == dst)
    v = g.views()
    assert np.array_equal(v[0], off) and np.array_equal(v[1], src) and v[2].tobytes() == cum.tobytes()
    assert np.array_equal(host.random_suspects_n(3000, 30, 2), g.random_suspects(30, 2))
    shell = host.Graph.shell(5, 7)
    assert (shell.n, shell.m) == (5, 7)


def test_multi_device_transport_selection(host):
    """host/multi.cpp: distinct devices go over NCCL (libnccl.so.2 is resolved at run time, all the
    entry points the solve calls are present), a repeated device id selects the in-process
    exchange (NCCL refuses duplicate devices), one device is the single-device path."""
    assert host.multi_transport([0, 1]) == "nccl"
    assert host.multi_transport([0, 1, 2, 3, 4, 5, 6, 7]) == "nccl"
    assert host.multi_transport([0, 0]) == "in-process exchange"
    assert host.multi_transport([3]) == "single device"

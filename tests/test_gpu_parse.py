"""Edge-list text ingest on the device: hsaw_gpu_edge_text_parse and
hsaw::load_edge_list_device against Python's correctly rounded float() (the value std::stod
returns), the host loader (reference-equivalent parser, tests/test_host_cpu.py pins it to the
reference) and the reference-generated fixture12 arrays. Lines outside the device parser's plain
grammar must be handed back, never guessed at (proj/src/graph.cpp:29-59, 201-263)."""
import os
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def _weight_strings(rng, count):
    out = []
    # what save_edge_list writes (graph.cpp:359: "%.17g") for weights in (0, 1]
    for x in rng.random(count // 4):
        out.append("%.17g" % (x if x > 0 else 0.5))
    for x in rng.random(count // 8):
        out.append(repr(float(x)))  # shortest round trip
    for _ in range(count // 8):  # short decimals
        out.append("%d.%0*d" % (rng.integers(0, 3), int(rng.integers(1, 8)), int(rng.integers(0, 10**7)) % 10 ** 7))
    for _ in range(count // 4):  # random significands and exponents, every digit count up to 19
        nd = int(rng.integers(1, 20))
        sig = int(rng.integers(10 ** (nd - 1), 10 ** nd - 1, dtype=np.uint64)) if nd > 1 else int(rng.integers(1, 10))
        e = int(rng.integers(-60, 40))
        form = int(rng.integers(0, 4))
        if form == 0:
            out.append(f"{sig}e{e}")
        elif form == 1:
            out.append(f"{sig}E{e:+d}")
        elif form == 2:
            s = str(sig)
            k = int(rng.integers(0, len(s)))
            out.append(f"{s[:k]}.{s[k:]}e{e}")
        else:
            out.append("0." + "0" * int(rng.integers(0, 12)) + str(sig))
    # exact binary fractions, halfway cases and their neighbours (round-to-even territory)
    for k in range(1, 40):
        out += [repr(2.0 ** -k), "%.17g" % (2.0 ** -k), str(2 ** 53 + 2 * k + 1), str(2 ** 53 + 2 * k)]
        out += [str((2 ** 53 + 2 * k + 1) * 10) + "e-1", str(2 ** 54 + 4 * k + 2)]
    out += ["9007199254740993", "9007199254740992", "9007199254740991", "1", "1.", ".5", "0", "0.0",
            "0e5", "00012.5000", "1e0", "1e22", "1e23", "8.5e22", "123456789012345678",
            "1234567890123456789", "4.9e-280", "1.7e270", "0.1", "0.2", "0.3", "1e-5"]
    while len(out) < count:
        out.append("%.17g" % rng.random())
    return out[:count]


def test_weights_are_the_correctly_rounded_doubles(gpu_lib):
    rng = np.random.Generator(np.random.PCG64(2024))
    ws = _weight_strings(rng, 400_000)
    text = "".join(f"{i} {i + 1} {w}\n" for i, w in enumerate(ws)).encode()
    with gpu_lib.Context(0) as ctx:
        r = ctx.parse_edge_text(text, weight_required=True, weight_values=True)
    assert r["host_line"] == 0, ws[r["host_line"] - 1]
    want = np.array([float(w) for w in ws])
    assert r["w"].size == want.size
    bad = np.flatnonzero(r["w"].view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, [(ws[i], r["w"][i], want[i]) for i in bad[:5]]
    assert r["identity"] and r["raw_ids"].size == len(ws) + 1
    assert np.array_equal(r["u"], np.arange(len(ws), dtype=np.uint32))


def test_lines_outside_the_plain_grammar_are_handed_back(gpu_lib):
    odd = ["-1 2", "+1 2", "1 2 -0.5", "1 2 +0.5", "1 2 0x1p-1", "1 2 inf", "1 2 nan", "1 2 1e-400",
           "1 2 1e400", "1 2 3 4", "1", "abc def", "1 2 1e", "1 2 .", "1 2 1.2.3", "1 2 1e5x",
           "12345678901234567890 1", "1 2 12345678901234567890123", "1 2x", "1 \x00 2",
           "1 2 0.1234567890123456789012"]
    with gpu_lib.Context(0) as ctx:
        for line in odd:
            text = ("0 1 0.5\n# c\n\n" + line + "\n7 8 0.25\n").encode("latin-1")
            r = ctx.parse_edge_text(text, weight_required=False)
            assert r["host_line"] == 4, line
        # a missing weight is only the host's business in given-weight mode (graph.cpp:216-218)
        text = b"0 1 0.5\n1 2\n"
        assert ctx.parse_edge_text(text, weight_required=True)["host_line"] == 2
        assert ctx.parse_edge_text(text, weight_required=False)["host_line"] == 0


def test_whitespace_comments_and_remap(gpu_lib):
    text = (b"# header\n"
            b"  \t 30 10 0.5 \r\n"
            b"\n"
            b"   # indented comment 1 2 3 4 5\n"
            b"\x0b\x0c 10\t\t20   0.25\n"
            b"20 30\n"
            b"007 30 1.\n"
            b"\r\n"
            b"1000000000000000000 7 .125")  # no trailing newline
    with gpu_lib.Context(0) as ctx:
        r = ctx.parse_edge_text(text)
        assert r["host_line"] == 0
        assert r["raw_ids"].tolist() == [7, 10, 20, 30, 10**18] and not r["identity"]
        assert r["u"].tolist() == [3, 1, 2, 0, 4] and r["v"].tolist() == [1, 2, 3, 3, 0]
        assert r["w"].tolist() == [0.5, 0.25, 0.0, 1.0, 0.125]
        for empty in (b"", b"\n", b"# only a comment", b"\n\n  \n"):
            r = ctx.parse_edge_text(empty)
            assert r["host_line"] == 0 and r["u"].size == 0
        r = ctx.parse_edge_text(b"0 1\n1 2\n2 0\n")
        assert r["identity"] and r["raw_ids"].tolist() == [0, 1, 2]


def _same_graph(a, b):
    for x, y in zip(a.arrays(), b.arrays()):
        assert x.dtype == y.dtype and np.array_equal(x.view(np.uint8), y.view(np.uint8))


def test_load_edge_list_device_equals_host_loader(tmp_path, golden):
    from paper_1702_05854_b200 import hostapi
    fx = golden["fixture12_given"]
    f12 = tmp_path / "fixture12.edges"
    with open(f12, "w") as f:
        f.write("# fixture12\n")
        for e in range(fx["m"]):
            f.write(f"{fx['in_src'][e]} {fx['edge_dst'][e]} {float.fromhex(fx['weight'][e])!r}\n")
    for mode in (0, 1, 2):
        a = hostapi.Graph.load_edge_list_device(f12, mode=mode, seed=5)
        _same_graph(a, hostapi.Graph.load_edge_list(f12, mode=mode, seed=5))
    g = hostapi.Graph.load_edge_list_device(f12, mode=0)
    off, src, cum, w, dst = g.arrays()  # the reference's own arrays for this file
    assert off.tolist() == fx["in_offsets"] and src.tolist() == fx["in_src"]
    assert [float.hex(float(x)) for x in cum] == fx["in_cum"]
    # what save_edge_list writes, every weight mode, ids that need the node map
    s = hostapi.Graph.synth(3000, 6, 11)
    p = tmp_path / "s.edges"
    s.save_edge_list(p)
    for mode in (0, 1):
        _same_graph(hostapi.Graph.load_edge_list_device(p, mode=mode),
                    hostapi.Graph.load_edge_list(p, mode=mode))
    lines = open(p).read().splitlines()
    q = tmp_path / "sparse_ids.edges"
    with open(q, "w") as f:
        for ln in lines:
            a, b, w = ln.split()
            f.write(f"{int(a) * 7 + 3}\t{int(b) * 7 + 3} {w}\n")
    dev = hostapi.Graph.load_edge_list_device(q, mode=0, mapping_out=tmp_path / "dev.map")
    host = hostapi.Graph.load_edge_list(q, mode=0, mapping_out=str(tmp_path / "host.map"))
    _same_graph(dev, host)
    assert open(tmp_path / "dev.map").read() == open(tmp_path / "host.map").read()
    # symmetrize is delegated to the host loader: same graph or same DataError
    def outcome(fn):
        try:
            return fn(q, mode=1, symmetrize=True).arrays()
        except hostapi.HsawError as e:
            return e.status, str(e)
    a, b = outcome(hostapi.Graph.load_edge_list_device), outcome(hostapi.Graph.load_edge_list)
    assert type(a) is type(b) and len(a) == len(b)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    tri = tmp_path / "tri.edges"
    tri.write_text("0 1\n1 2\n2 0\n")
    _same_graph(hostapi.Graph.load_edge_list_device(tri, mode=1, symmetrize=True),
                hostapi.Graph.load_edge_list(tri, mode=1, symmetrize=True))


def test_error_files_raise_what_the_host_loader_raises(tmp_path):
    from paper_1702_05854_b200 import hostapi
    cases = {
        "malformed": "0 1 0.5\n1 2 zebra\n",
        "trailing": "0 1 0.5 9\n",
        "weight_required": "0 1 0.5\n1 2\n",
        "duplicate": "0 1 0.5\n0 1 0.25\n",
        "self_loop": "0 1 0.5\n2 2 0.5\n",
        "weight_range": "0 1 0.5\n1 2 1.5\n",
        "zero_weight": "0 1 0\n",
        "sum_above_one": "0 2 0.75\n1 2 0.75\n",
        "negative_id": "0 1 0.5\n-1 2 0.5\n",
        "empty": "",
        "only_comments": "# nothing\n\n",
    }
    for name, body in cases.items():
        p = tmp_path / (name + ".edges")
        p.write_text(body)
        for mode in (0, 1):
            try:
                want = ("ok", hostapi.Graph.load_edge_list(p, mode=mode).arrays())
            except hostapi.HsawError as e:
                want = (e.status, str(e))
            try:
                got = ("ok", hostapi.Graph.load_edge_list_device(p, mode=mode).arrays())
            except hostapi.HsawError as e:
                got = (e.status, str(e))
            if want[0] == "ok":
                assert got[0] == "ok", (name, mode, got)
                for x, y in zip(want[1], got[1]):
                    assert np.array_equal(x, y)
            else:
                assert got == want, (name, mode)
    with pytest.raises(hostapi.HsawError) as ei:
        hostapi.Graph.load_edge_list_device(tmp_path / "missing.edges")
    assert ei.value.status == 2 and "cannot open edge list" in str(ei.value)


def test_full_size_text_round_trip(tmp_path):
    """C2 shape: 16 M lines written by save_edge_list, read back in 1/in-degree mode."""
    from paper_1702_05854_b200 import hostapi
    g = hostapi.Graph.rmat(20, 16.0, seed=1)
    p = tmp_path / "c2.edges"
    g.save_edge_list(p)
    assert os.path.getsize(p) > 300e6
    try:
        back = hostapi.Graph.load_edge_list_device(p, mode=1)
    except hostapi.HsawError as e:  # validate() may reject R-MAT hub rows
        assert e.status == 2 and "in-weight sum" in str(e)
        return
    off, src, cum, _, dst = g.arrays()
    boff, bsrc, bcum, _, bdst = back.arrays()
    # nodes without any edge do not appear in the file: ids are re-ranked (graph.cpp:222-241)
    present = np.unique(np.concatenate([src, dst]))
    assert back.n == present.size and back.m == g.m
    assert np.array_equal(bsrc, np.searchsorted(present, src).astype(np.uint32))
    assert np.array_equal(bdst, np.searchsorted(present, dst).astype(np.uint32))
    assert boff[0] == 0 and np.array_equal(boff[1:], off[present.astype(np.int64) + 1])
    assert np.array_equal(cum.view(np.uint64), bcum.view(np.uint64))


def test_text_to_resident_graph_without_host_csr(tmp_path, gpu_lib):
    """DeviceGraph::from_edge_list / hsaw_gpu_edge_text_install: the parsed edges are sorted,
    summed and laid out where they lie on the device; sampling equals the host-loaded graph's."""
    from paper_1702_05854_b200 import hostapi
    s = hostapi.Graph.synth(3000, 6, 11)
    p = tmp_path / "s.edges"
    s.save_edge_list(p)
    for mode in (0, 1):
        g = hostapi.Graph.load_edge_list(p, mode=mode)
        p_of = g.random_suspects(30, seed=4)
        with hostapi.DeviceGraph(g, p_of) as dg:
            want = dg.sample(2000, seed=5)
            est = hostapi.estimate_suspension(g, p_of, 0, [3, 4, 5], 0.3, 0.2, 9, dg=dg)
        dg = hostapi.DeviceGraph.from_edge_list(p, mode=mode)
        assert dg is not None
        with dg:
            dg.set_suspects(g, p_of)
            assert dg.sample(2000, seed=5) == want
            assert hostapi.estimate_suspension(g, p_of, 0, [3, 4, 5], 0.3, 0.2, 9, dg=dg) == est
    # outside the plain grammar / host-only modes: no device graph, the host loader decides
    odd = tmp_path / "odd.edges"
    odd.write_text("0 1 0.5\n1 2 +0.25\n")
    assert hostapi.DeviceGraph.from_edge_list(odd, mode=0) is None
    assert hostapi.DeviceGraph.from_edge_list(p, mode=2) is None
    # data errors surface with build_graph's messages
    dup = tmp_path / "dup.edges"
    dup.write_text("0 1 0.5\n0 1 0.25\n")
    with pytest.raises(hostapi.HsawError) as ei:
        hostapi.DeviceGraph.from_edge_list(dup, mode=0)
    assert ei.value.status == 2 and "duplicate edge 0 -> 1" in str(ei.value)
    with gpu_lib.Context(0) as ctx:
        assert ctx.upload_edge_text(b"5 7\n7 9\n9 5\n", weight_mode=1,
                                    p_of=np.array([1.0, 0.0, 0.0])) == (3, 3)
        seeds, lens, counts, _ = ctx.encode_batches(0, 4)
        assert counts.sum() > 0

"""Generates tests/golden/cache_vectors.npz + cache_errors.json with the UNMODIFIED reference
(oracle/_ref): HSAW1 images written by the reference's save_cache, the arrays its load_cache
returns for them, and the DataError messages it raises for corrupted images (only corruptions that
keep the reference's own loops in bounds). Usage:  python tests/golden/make_cache_golden.py
"""
import json
import os
import struct
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import OracleError, Ref  # noqa: E402


def arrays(R, gh):
    csr = R._to_csr(gh)
    w, dst = R.graph_extra(gh)
    return csr.in_offsets, csr.in_src, csr.in_cum, w, dst


def patch_u64(img: bytearray, word: int, value: int):
    img[21 + 8 * word: 29 + 8 * word] = struct.pack("<Q", value)


def patch_f64(img: bytearray, word: int, value: float):
    img[21 + 8 * word: 29 + 8 * word] = struct.pack("<d", value)


def main():
    R = Ref()
    out, errors = {}, {}
    with tempfile.TemporaryDirectory() as tmp:
        graphs = {
            "fixture12": R.load_edge_list("/root/reference/proj/data/fixture12.edges", mode=0),
            "synth300": R.synth_graph(300, 5, 21),
            "synth2000_random": None,
        }
        # random-normalized weights: rows that do not sum to exactly 1
        g0 = R.synth_graph(2000, 4, 9)
        c0 = R._to_csr(g0)
        _, d0 = R.graph_extra(g0)
        graphs["synth2000_random"] = R.build_graph(2000, c0.in_src, d0, None, mode=2, seed=77)
        for name, gh in graphs.items():
            path = os.path.join(tmp, name + ".hsaw1")
            R.save_cache(gh, path)
            img = open(path, "rb").read()
            back = R.load_cache(path)
            off, src, cum, w, dst = arrays(R, back)
            out[name + "_image"] = np.frombuffer(img, dtype=np.uint8)
            for k, a in zip(("off", "src", "cum", "weight", "dst"), (off, src, cum, w, dst)):
                out[f"{name}_{k}"] = a

        # corrupted images of synth300 and the reference's message for each
        img0 = bytes(out["synth300_image"].tobytes())
        n, m = struct.unpack("<QQ", img0[5:21])
        off = out["synth300_off"]
        v = int(np.flatnonzero(np.diff(off.astype(np.int64)) >= 3)[5])  # a row with >= 3 edges
        lo = int(off[v])
        src_word, w_word = n + 1 + lo, n + 1 + m + lo
        cases = {}
        b = bytearray(img0); b[0:5] = b"HSAWX"; cases["bad_magic"] = bytes(b)
        cases["truncated"] = img0[:-9]
        cases["header_only"] = img0[:21]
        b = bytearray(img0); patch_u64(b, src_word + 1, n + 7); cases["source_out_of_range"] = bytes(b)
        b = bytearray(img0); patch_u64(b, src_word, v); cases["self_loop"] = bytes(b)
        b = bytearray(img0); patch_u64(b, src_word + 1, int(out["synth300_src"][lo])); cases["duplicate"] = bytes(b)
        b = bytearray(img0); patch_f64(b, w_word + 1, 0.0); cases["zero_weight"] = bytes(b)
        b = bytearray(img0); patch_f64(b, w_word + 2, 1.5); cases["weight_above_one"] = bytes(b)
        b = bytearray(img0); patch_f64(b, w_word + 1, float("nan")); cases["nan_weight"] = bytes(b)
        b = bytearray(img0); patch_f64(b, w_word, 0.9); patch_f64(b, w_word + 1, 0.9); cases["row_sum_above_one"] = bytes(b)
        b = bytearray(img0); patch_f64(b, w_word, 1.0); patch_f64(b, w_word + 1, 1e-300); cases["cum_not_increasing"] = bytes(b)
        b = bytearray(img0); patch_u64(b, 0, 1); cases["first_offset_nonzero"] = bytes(b)
        # two errors in different rows: the lower row wins whatever its kind
        v2 = int(np.flatnonzero(np.diff(off.astype(np.int64)) >= 3)[20])
        b = bytearray(img0); patch_f64(b, n + 1 + m + int(off[v2]), 2.0); patch_u64(b, src_word, v); cases["two_rows"] = bytes(b)
        for name, data in cases.items():
            path = os.path.join(tmp, name + ".hsaw1")
            open(path, "wb").write(data)
            try:
                R.load_cache(path)
                msg = None
            except OracleError as e:
                msg = str(e).split("load_cache: ", 1)[1].replace(path, "<path>")
                assert e.status == 2, (name, e.status)
            errors[name] = msg
            out["bad_" + name] = np.frombuffer(data, dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "cache_vectors.npz"), **out)
    json.dump(errors, open(os.path.join(HERE, "cache_errors.json"), "w"), indent=1)
    print(json.dumps(errors, indent=1))


if __name__ == "__main__":
    main()

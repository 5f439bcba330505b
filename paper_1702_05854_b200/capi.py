"""ctypes binding of include/hsaw_gpu.h (plumbing for tests/ and bench.py — not the product).

The product is the shared library; this module only marshals numpy arrays into its C-ABI. There is
no fallback of any kind: a missing library or a missing CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _build

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
u8p = C.POINTER(C.c_uint8)
f64p = C.POINTER(C.c_double)

HSAW_OK, HSAW_EINVAL, HSAW_EDATA, HSAW_EBUDGET, HSAW_ERANGE, HSAW_ECUDA = range(6)
KIND_EDGE, KIND_NODE = 0, 1

STAGE_NAMES = ("encode", "decode", "distinct", "compact", "index", "rounds", "coverage", "upload",
               "simulate")
STAT_NAMES = ("attempts", "draws", "steps", "alg_bytes", "accepted", "decode_steps", "dropped",
              "spare")


class HsawError(RuntimeError):
    """Mirrors the reference's exception -> exit-code mapping (proj/src/cli.cpp:520-538)."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"hsaw_gpu status {status}: {msg}")
        self.status = status
        self.msg = msg


class SamplerCfg(C.Structure):
    """hsaw_sampler_cfg == SamplerConfig (proj/include/hsaw/sampler.hpp:48-55)."""

    _fields_ = [("heuristic", C.c_int32), ("window", C.c_uint32), ("batch_size", C.c_uint32),
                ("max_attempts", C.c_uint64), ("rng_mode", C.c_uint32)]

    def __init__(self, heuristic=0, window=2, batch_size=10, max_attempts=100_000_000, rng_mode=0):
        """rng_mode 0: the reference's stream (bit-exact); 1: Philox per-walk throughput mode."""
        super().__init__(heuristic, window, batch_size, max_attempts, rng_mode)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


_LIB = None


def lib() -> C.CDLL:
    """Loads libhsaw_gpu.so from the package tree (never from site-packages, never rebuilt here)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(_build.GPU_SO):
        raise ImportError(
            f"{_build.GPU_SO} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback for this path.")
    L = C.CDLL(_build.GPU_SO)
    vp = C.c_void_p
    L.hsaw_gpu_ctx_create.argtypes = [C.c_int, vp, C.POINTER(vp)]
    L.hsaw_gpu_ctx_destroy.argtypes = [vp]
    L.hsaw_gpu_ctx_destroy.restype = None
    L.hsaw_gpu_last_error.argtypes = [vp]
    L.hsaw_gpu_last_error.restype = C.c_char_p
    L.hsaw_gpu_ctx_cuda_stream.argtypes = [vp]
    L.hsaw_gpu_ctx_cuda_stream.restype = vp
    L.hsaw_gpu_ctx_sync.argtypes = [vp]
    L.hsaw_gpu_graph_upload.argtypes = [vp, C.c_uint32, C.c_uint32, u64p, u32p, f64p, f64p]
    L.hsaw_gpu_suspects_upload.argtypes = [vp, f64p]
    L.hsaw_gpu_csr_build.argtypes = [vp, C.c_uint32, C.c_uint64, u32p, u32p, f64p, C.c_int, u64p,
                                     u32p, f64p, f64p, u32p]
    L.hsaw_gpu_graph_build_upload.argtypes = [vp, C.c_uint32, C.c_uint64, u32p, u32p, f64p,
                                              C.c_int, f64p]
    L.hsaw_gpu_cache_decode.argtypes = [vp, C.c_uint32, C.c_uint32, vp, u64p, u32p, f64p, f64p, u32p]
    L.hsaw_gpu_graph_cache_upload.argtypes = [vp, C.c_uint32, C.c_uint32, vp, f64p]
    L.hsaw_gpu_edge_text_parse.argtypes = [vp, C.c_char_p, C.c_uint64, C.c_int, C.c_int,
                                           C.POINTER(vp), u64p, u64p, C.POINTER(C.c_int), u64p]
    L.hsaw_gpu_edge_text_fetch.argtypes = [vp, u32p, u32p, f64p, u64p]
    L.hsaw_gpu_edge_text_install.argtypes = [vp, C.c_int, f64p]
    L.hsaw_gpu_edge_text_free.argtypes = [vp]
    L.hsaw_gpu_edge_text_free.restype = None
    L.hsaw_gpu_graph_bytes.argtypes = [vp]
    L.hsaw_gpu_graph_bytes.restype = C.c_uint64
    L.hsaw_gpu_graph_layout.argtypes = [vp]
    L.hsaw_gpu_graph_upload_mode.argtypes = [vp]
    L.hsaw_gpu_graph_upload_bytes.argtypes = [vp]
    L.hsaw_gpu_graph_upload_bytes.restype = C.c_uint64
    L.hsaw_gpu_launch_count.argtypes = [vp]
    L.hsaw_gpu_launch_count.restype = C.c_uint64
    L.hsaw_gpu_stage_times.argtypes = [vp, f64p, u64p, C.c_int]
    L.hsaw_gpu_debug_counters.argtypes = [f64p]
    L.hsaw_gpu_debug_counters.restype = None
    L.hsaw_gpu_encode_batches.argtypes = [vp, C.POINTER(SamplerCfg), C.c_uint64, C.c_uint64, u64p,
                                          u32p, u32p, u64p]
    L.hsaw_gpu_encode_stats.argtypes = [vp, C.POINTER(SamplerCfg), C.c_uint64, C.c_uint64, u64p]
    L.hsaw_gpu_decode_walks.argtypes = [vp, C.c_uint64, u64p, u32p, u64p, u32p, u32p, u8p]
    L.hsaw_gpu_stream_create.argtypes = [vp, C.c_uint64, C.POINTER(SamplerCfg), C.POINTER(vp)]
    L.hsaw_gpu_stream_keep.argtypes = [vp, C.c_int, C.c_int]
    L.hsaw_gpu_stream_restrict.argtypes = [vp, u32p, C.c_uint64, C.POINTER(C.c_uint8)]
    L.hsaw_gpu_stream_crossings.argtypes = [vp, C.c_uint64, u64p]
    L.hsaw_gpu_stream_destroy.argtypes = [vp]
    L.hsaw_gpu_stream_destroy.restype = None
    L.hsaw_gpu_stream_ensure.argtypes = [vp, C.c_uint64]
    L.hsaw_gpu_stream_sample_range.argtypes = [vp, C.c_uint64, C.c_uint64, u64p]
    L.hsaw_gpu_stream_size.argtypes = [vp, u64p, u64p, u64p]
    L.hsaw_gpu_stream_counters.argtypes = [vp, C.c_uint64, u64p, u64p]
    L.hsaw_gpu_stream_local_cut.argtypes = [vp, C.c_uint64, u64p, u64p]
    L.hsaw_gpu_stream_slice_edges.argtypes = [vp, C.c_uint64, C.c_uint64, u64p]
    L.hsaw_gpu_stream_export.argtypes = [vp, C.c_uint64, C.c_uint64, u64p, u32p, u32p, u64p, u32p]
    L.hsaw_gpu_stream_stats.argtypes = [vp, u64p]
    L.hsaw_gpu_stream_collect_stats.argtypes = [vp, C.c_int]
    L.hsaw_gpu_walkset_import.argtypes = [vp, C.c_uint32, C.c_uint64, u64p, u32p, C.POINTER(vp)]
    L.hsaw_gpu_walkset_destroy.argtypes = [vp]
    L.hsaw_gpu_walkset_destroy.restype = None
    L.hsaw_gpu_greedy.argtypes = [vp, vp, vp, C.c_int, C.c_uint64, C.c_uint64, u32p, C.c_uint64,
                                  C.c_uint32, u32p, u64p]
    L.hsaw_gpu_coverage_of.argtypes = [vp, vp, vp, C.c_int, C.c_uint64, C.c_uint64, u32p,
                                       C.c_uint64, u32p, C.c_uint64, u64p]
    L.hsaw_gpu_coverage_upper_bound.argtypes = [vp, vp, vp, C.c_int, C.c_uint64, C.c_uint64, u32p,
                                                C.c_uint64, C.c_uint32, u64p]
    L.hsaw_gpu_rounds_begin.argtypes = [vp, vp, vp, C.c_int, C.c_uint64, C.c_uint64, u32p,
                                        C.c_uint64, vp, C.POINTER(vp)]
    L.hsaw_gpu_rounds_occurrences.argtypes = [vp]
    L.hsaw_gpu_rounds_occurrences.restype = C.c_uint64
    L.hsaw_gpu_rounds_select.argtypes = [vp, u32p, u64p]
    L.hsaw_gpu_rounds_cover.argtypes = [vp, C.c_uint32, vp, C.c_uint64, u64p]
    L.hsaw_gpu_rounds_apply.argtypes = [vp, vp, C.c_uint64]
    L.hsaw_gpu_rounds_end.argtypes = [vp]
    L.hsaw_gpu_rounds_end.restype = None
    L.hsaw_gpu_paired_runs.argtypes = [vp, C.c_int, u32p, C.c_uint64, u64p, C.c_uint64, u32p, u32p]
    L.hsaw_gpu_rr_node_sets.argtypes = [vp, u64p, C.c_uint32, C.POINTER(vp), u64p]
    L.hsaw_gpu_walkset_export.argtypes = [vp, u64p, u32p]
    L.hsaw_gpu_stream_histogram.argtypes = [vp, vp, C.c_int, C.c_uint64, C.c_uint64, u32p, C.c_uint64, vp]
    L.hsaw_gpu_counts_bound.argtypes = [vp, vp, C.c_uint32, C.c_uint32, C.c_uint64, u64p]
    L.hsaw_gpu_counts_threshold.argtypes = [vp, vp, C.c_uint32, u32p]
    L.hsaw_gpu_counts_threshold_for.argtypes = [vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, u32p]
    L.hsaw_gpu_reduced_walks.argtypes = [vp, vp, C.c_int, C.c_uint64, C.c_uint64, vp, C.c_uint32,
                                         C.POINTER(vp), u64p, u64p]
    L.hsaw_gpu_walkset_copy_device.argtypes = [vp, vp, vp]
    L.hsaw_gpu_walkset_from_device.argtypes = [vp, C.c_uint32, C.c_uint64, vp, vp, C.c_uint64,
                                               C.POINTER(vp)]
    L.hsaw_gpu_last_greedy_min_gain.argtypes = [vp]
    L.hsaw_gpu_last_greedy_min_gain.restype = C.c_uint64
    L.hsaw_gpu_prg_jump.argtypes = [C.c_uint64, C.c_uint64]
    L.hsaw_gpu_prg_jump.restype = C.c_uint64
    L.hsaw_gpu_estimate_suspension.argtypes = [vp, C.c_int, u32p, C.c_uint64, C.c_double,
                                               C.c_double, u64p, f64p, C.POINTER(C.c_int), u64p]
    _LIB = L
    return L


# Every symbol include/hsaw_gpu.h declares (checked by the CPU test-suite against the built .so).
EXPORTS = (
    "hsaw_gpu_ctx_create", "hsaw_gpu_ctx_destroy", "hsaw_gpu_last_error",
    "hsaw_gpu_ctx_cuda_stream", "hsaw_gpu_ctx_sync", "hsaw_gpu_graph_upload",
    "hsaw_gpu_csr_build", "hsaw_gpu_graph_build_upload",
    "hsaw_gpu_suspects_upload", "hsaw_gpu_graph_bytes", "hsaw_gpu_encode_batches",
    "hsaw_gpu_encode_stats",
    "hsaw_gpu_decode_walks", "hsaw_gpu_stream_create", "hsaw_gpu_stream_destroy",
    "hsaw_gpu_stream_ensure", "hsaw_gpu_stream_sample_range", "hsaw_gpu_stream_size",
    "hsaw_gpu_stream_counters", "hsaw_gpu_stream_local_cut", "hsaw_gpu_stream_slice_edges",
    "hsaw_gpu_stream_export", "hsaw_gpu_stream_stats", "hsaw_gpu_stream_collect_stats", "hsaw_gpu_walkset_import",
    "hsaw_gpu_walkset_destroy", "hsaw_gpu_greedy", "hsaw_gpu_coverage_of",
    "hsaw_gpu_coverage_upper_bound",
    "hsaw_gpu_launch_count", "hsaw_gpu_stage_times", "hsaw_gpu_debug_counters",
    "hsaw_gpu_rounds_begin", "hsaw_gpu_rounds_occurrences", "hsaw_gpu_rounds_select",
    "hsaw_gpu_rounds_cover", "hsaw_gpu_rounds_apply", "hsaw_gpu_rounds_end",
    "hsaw_gpu_paired_runs", "hsaw_gpu_estimate_suspension",
    "hsaw_gpu_cache_decode", "hsaw_gpu_graph_cache_upload", "hsaw_gpu_prg_jump",
    "hsaw_gpu_edge_text_parse", "hsaw_gpu_edge_text_fetch", "hsaw_gpu_edge_text_free",
    "hsaw_gpu_edge_text_install",
    "hsaw_gpu_rmat_build", "hsaw_gpu_held_csr_fetch", "hsaw_gpu_held_csr_install",
    "hsaw_gpu_held_csr_drop", "hsaw_gpu_graph_layout", "hsaw_gpu_graph_upload_mode", "hsaw_gpu_graph_upload_bytes",
    "hsaw_gpu_stream_keep",
    "hsaw_gpu_stream_restrict", "hsaw_gpu_stream_crossings",
    "hsaw_gpu_rr_node_sets", "hsaw_gpu_walkset_export",
    "hsaw_gpu_stream_histogram", "hsaw_gpu_counts_bound", "hsaw_gpu_counts_threshold",
    "hsaw_gpu_counts_threshold_for",
    "hsaw_gpu_reduced_walks", "hsaw_gpu_walkset_copy_device", "hsaw_gpu_walkset_from_device",
    "hsaw_gpu_last_greedy_min_gain", "hsaw_gpu_device_alloc", "hsaw_gpu_device_free",
    "hsaw_gpu_device_copy", "hsaw_gpu_counts_add",
)


def prg_jump(state: int, draws: int) -> int:
    """PrgState.state after `draws` xorshift64* steps (GF(2) jump-ahead; host arithmetic only)."""
    return int(lib().hsaw_gpu_prg_jump(state, draws))


def alloc_counters() -> dict:
    out = np.zeros(3, dtype=np.float64)
    lib().hsaw_gpu_debug_counters(_p(out, f64p))
    return dict(seconds=float(out[0]), calls=int(out[1]), bytes=int(out[2]))


@dataclass
class Pool:
    """Host copy of a stream slice, same layout as the oracle's PoolData."""

    attempts: int
    edge_off: np.ndarray
    nodes: np.ndarray
    edges: np.ndarray
    tag_worker: np.ndarray
    tag_seq: np.ndarray

    @property
    def nsamples(self) -> int:
        return len(self.edge_off) - 1

    def walk_nodes(self, w):
        return self.nodes[int(self.edge_off[w]) + w: int(self.edge_off[w + 1]) + w + 1]

    def walk_edges(self, w):
        return self.edges[int(self.edge_off[w]): int(self.edge_off[w + 1])]


class Context:
    """hsaw_gpu_ctx: one device + the uploaded graph."""

    def __init__(self, device: int = 0, cuda_stream: int | None = None):
        self.L = lib()
        self.h = C.c_void_p()
        rc = self.L.hsaw_gpu_ctx_create(device, C.c_void_p(cuda_stream) if cuda_stream else None,
                                        C.byref(self.h))
        if rc != HSAW_OK:
            raise HsawError(rc, "hsaw_gpu_ctx_create failed: no usable CUDA device "
                                "(this path has no CPU fallback)")
        self.n = self.m = 0

    @classmethod
    def borrow(cls, handle, n=0, m=0) -> "Context":
        """Non-owning view of an existing hsaw_gpu_ctx* (e.g. the one inside a DeviceGraph)."""
        self = cls.__new__(cls)
        self.L = lib()
        self.h = C.c_void_p(handle)
        self.n, self.m = n, m
        self._borrowed = True
        return self

    def close(self):
        if self.h and not getattr(self, "_borrowed", False):
            self.L.hsaw_gpu_ctx_destroy(self.h)
        self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _chk(self, rc):
        if rc != HSAW_OK:
            raise HsawError(rc, self.L.hsaw_gpu_last_error(self.h).decode())

    def sync(self):
        self._chk(self.L.hsaw_gpu_ctx_sync(self.h))

    @property
    def cuda_stream(self) -> int:
        return int(self.L.hsaw_gpu_ctx_cuda_stream(self.h) or 0)

    @property
    def launches(self) -> int:
        return int(self.L.hsaw_gpu_launch_count(self.h))

    def stage_times(self, reset: bool = False) -> dict:
        """{stage: (ms, timed regions)} measured with CUDA events around the kernels."""
        ms = np.zeros(len(STAGE_NAMES), dtype=np.float64)
        cnt = np.zeros(len(STAGE_NAMES), dtype=np.uint64)
        self._chk(self.L.hsaw_gpu_stage_times(self.h, _p(ms, f64p), _p(cnt, u64p), int(reset)))
        return {n: (float(ms[i]), int(cnt[i])) for i, n in enumerate(STAGE_NAMES)}

    # -- paired LT forward simulation (proj/src/evaluation.cpp:49-108,202-242)
    def paired_runs(self, kind, ids, state, nruns):
        """-> (full u32[nruns], residual u32[nruns], state_after). kind -1: no removal."""
        a = np.ascontiguousarray([] if ids is None else ids, dtype=np.uint32)
        buf = a if a.size else np.zeros(1, dtype=np.uint32)
        full = np.zeros(max(nruns, 1), dtype=np.uint32)
        res = np.zeros(max(nruns, 1), dtype=np.uint32)
        s = C.c_uint64(state)
        self._chk(self.L.hsaw_gpu_paired_runs(self.h, kind, _p(buf, u32p), a.size, C.byref(s),
                                              nruns, _p(full, u32p), _p(res, u32p)))
        return full[:nruns], res[:nruns], s.value

    def lt_forward_simulate(self, state):
        """lt_forward_simulate(g, vi, s): -> (infected, state_after)."""
        full, _, after = self.paired_runs(-1, None, state, 1)
        return int(full[0]), after

    def estimate_suspension(self, kind, ids, eps, delta, state):
        """-> dict(value, capped, runs, state) like SuspensionEstimate + the advanced PrgState."""
        a = np.ascontiguousarray(ids, dtype=np.uint32)
        buf = a if a.size else np.zeros(1, dtype=np.uint32)
        s, v, cp, runs = C.c_uint64(state), C.c_double(), C.c_int(), C.c_uint64()
        self._chk(self.L.hsaw_gpu_estimate_suspension(self.h, kind, _p(buf, u32p), a.size, eps,
                                                      delta, C.byref(s), C.byref(v), C.byref(cp),
                                                      C.byref(runs)))
        return dict(value=v.value, capped=bool(cp.value), runs=int(runs.value), state=s.value)

    @property
    def graph_bytes(self) -> int:
        return int(self.L.hsaw_gpu_graph_bytes(self.h))

    @property
    def graph_layout(self) -> str:
        code = int(self.L.hsaw_gpu_graph_layout(self.h))
        return {0: "fat", -1: "none"}.get(code, "compact")

    @property
    def upload_mode(self) -> str:
        return "regenerated" if int(self.L.hsaw_gpu_graph_upload_mode(self.h)) == 1 else "copied"

    @property
    def upload_bytes(self) -> int:
        return int(self.L.hsaw_gpu_graph_upload_bytes(self.h))

    def upload_graph(self, n, m, in_offsets, in_src, in_cum, p_of):
        in_offsets = np.ascontiguousarray(in_offsets, dtype=np.uint64)
        in_src = np.ascontiguousarray(in_src, dtype=np.uint32)
        in_cum = np.ascontiguousarray(in_cum, dtype=np.float64)
        p_of = np.ascontiguousarray(p_of, dtype=np.float64)
        assert in_offsets.shape == (n + 1,) and in_src.shape == (m,) and in_cum.shape == (m,)
        assert p_of.shape == (n,)
        self._chk(self.L.hsaw_gpu_graph_upload(self.h, n, m, _p(in_offsets, u64p),
                                               _p(in_src, u32p), _p(in_cum, f64p), _p(p_of, f64p)))
        self.n, self.m = n, m

    def parse_edge_text(self, text: bytes, weight_required=False, weight_values=True):
        """Device half of load_edge_list: -> dict(u, v, w, raw_ids, identity) or dict(host_line=N)
        when line N is outside the plain grammar and the host parser must take over."""
        h = C.c_void_p()
        ne, nids, ident, hl = C.c_uint64(), C.c_uint64(), C.c_int(), C.c_uint64()
        self._chk(self.L.hsaw_gpu_edge_text_parse(self.h, text, len(text), int(weight_required),
                                                  int(weight_values), C.byref(h), C.byref(ne),
                                                  C.byref(nids), C.byref(ident), C.byref(hl)))
        if hl.value:
            return dict(host_line=int(hl.value))
        ne, nids = ne.value, nids.value
        u = np.zeros(max(ne, 1), dtype=np.uint32)
        v = np.zeros(max(ne, 1), dtype=np.uint32)
        w = np.zeros(max(ne, 1), dtype=np.float64)
        ids = np.zeros(max(nids, 1), dtype=np.uint64)
        if h:
            try:
                self._chk(self.L.hsaw_gpu_edge_text_fetch(h, _p(u, u32p), _p(v, u32p),
                                                          _p(w, f64p), _p(ids, u64p)))
            finally:
                self.L.hsaw_gpu_edge_text_free(h)
        return dict(u=u[:ne], v=v[:ne], w=w[:ne], raw_ids=ids[:nids], identity=bool(ident.value),
                    host_line=0)

    def upload_edge_text(self, text: bytes, weight_mode=1, p_of=None):
        """Edge-list text -> graph resident and ready to sample (no host CSR). Returns (n, m), or
        None when a line is outside the device parser's plain grammar (host loader's business)."""
        h = C.c_void_p()
        ne, nids, ident, hl = C.c_uint64(), C.c_uint64(), C.c_int(), C.c_uint64()
        given = weight_mode == 0
        self._chk(self.L.hsaw_gpu_edge_text_parse(self.h, text, len(text), int(given), int(given),
                                                  C.byref(h), C.byref(ne), C.byref(nids),
                                                  C.byref(ident), C.byref(hl)))
        if hl.value or not h:
            return None
        try:
            p = None if p_of is None else np.ascontiguousarray(p_of, dtype=np.float64)
            self._chk(self.L.hsaw_gpu_edge_text_install(h, weight_mode,
                                                        _p(p, f64p) if p is not None else None))
        finally:
            self.L.hsaw_gpu_edge_text_free(h)
        self.n, self.m = int(nids.value), int(ne.value)
        return self.n, self.m

    @staticmethod
    def _cache_header(image: bytes):
        """(n, m) from an HSAW1 image (graph.cpp:398-405); the host layer owns the file errors."""
        if len(image) < 21 or image[:5] != b"HSAW1":
            raise HsawError(HSAW_EDATA, "bad cache magic")
        n = int.from_bytes(image[5:13], "little") & 0xFFFFFFFF
        m = int.from_bytes(image[13:21], "little") & 0xFFFFFFFF
        if len(image) < 21 + 8 * (n + 1 + 2 * m):
            raise HsawError(HSAW_EDATA, "truncated cache")
        return n, m

    def decode_cache(self, image: bytes, aux=True):
        """load_cache on the device: (in_offsets, in_src, in_cum, weight, edge_dst) host arrays."""
        n, m = self._cache_header(image)
        buf = np.frombuffer(image, dtype=np.uint8)
        off = np.zeros(n + 1, dtype=np.uint64)
        src = np.zeros(max(m, 1), dtype=np.uint32)
        cum = np.zeros(max(m, 1), dtype=np.float64)
        wt = np.zeros(max(m, 1), dtype=np.float64) if aux else None
        dst = np.zeros(max(m, 1), dtype=np.uint32) if aux else None
        self._chk(self.L.hsaw_gpu_cache_decode(
            self.h, n, m, C.c_void_p(buf.ctypes.data + 21), _p(off, u64p), _p(src, u32p),
            _p(cum, f64p), _p(wt, f64p) if aux else None, _p(dst, u32p) if aux else None))
        return off, src[:m], cum[:m], (wt[:m] if aux else None), (dst[:m] if aux else None)

    def upload_cache(self, image: bytes, p_of=None):
        """HSAW1 image -> graph resident and ready to sample, no host CSR."""
        n, m = self._cache_header(image)
        buf = np.frombuffer(image, dtype=np.uint8)
        p = None if p_of is None else np.ascontiguousarray(p_of, dtype=np.float64)
        self._chk(self.L.hsaw_gpu_graph_cache_upload(self.h, n, m, C.c_void_p(buf.ctypes.data + 21),
                                                     _p(p, f64p) if p is not None else None))
        self.n, self.m = n, m

    def build_csr(self, n, edge_u, edge_v, edge_w=None, weight_mode=1, aux=True):
        """build_graph on the device (proj/src/graph.cpp:112-199): returns (in_offsets, in_src,
        in_cum, weight, edge_dst) as host arrays. weight_mode 0 Given, 1 InDegree."""
        edge_u = np.ascontiguousarray(edge_u, dtype=np.uint32)
        edge_v = np.ascontiguousarray(edge_v, dtype=np.uint32)
        ne = int(edge_u.size)
        assert edge_v.shape == (ne,)
        w = None if edge_w is None else np.ascontiguousarray(edge_w, dtype=np.float64)
        off = np.zeros(n + 1, dtype=np.uint64)
        src = np.zeros(ne, dtype=np.uint32)
        cum = np.zeros(ne, dtype=np.float64)
        wt = np.zeros(ne, dtype=np.float64) if aux else None
        dst = np.zeros(ne, dtype=np.uint32) if aux else None
        self._chk(self.L.hsaw_gpu_csr_build(
            self.h, n, ne, _p(edge_u, u32p), _p(edge_v, u32p), _p(w, f64p) if w is not None else None,
            weight_mode, _p(off, u64p), _p(src, u32p), _p(cum, f64p),
            _p(wt, f64p) if aux else None, _p(dst, u32p) if aux else None))
        return off, src, cum, wt, dst

    def build_upload_graph(self, n, edge_u, edge_v, p_of, edge_w=None, weight_mode=1):
        """Edge list -> device graph without a host CSR (hsaw_gpu_graph_build_upload)."""
        edge_u = np.ascontiguousarray(edge_u, dtype=np.uint32)
        edge_v = np.ascontiguousarray(edge_v, dtype=np.uint32)
        p_of = np.ascontiguousarray(p_of, dtype=np.float64)
        ne = int(edge_u.size)
        w = None if edge_w is None else np.ascontiguousarray(edge_w, dtype=np.float64)
        self._chk(self.L.hsaw_gpu_graph_build_upload(
            self.h, n, ne, _p(edge_u, u32p), _p(edge_v, u32p),
            _p(w, f64p) if w is not None else None, weight_mode, _p(p_of, f64p)))
        self.n, self.m = n, ne

    def upload_suspects(self, p_of):
        p_of = np.ascontiguousarray(p_of, dtype=np.float64)
        assert p_of.shape == (self.n,)
        self._chk(self.L.hsaw_gpu_suspects_upload(self.h, _p(p_of, f64p)))

    # ---- K1 / K2 parity entry points
    def encode_batches(self, first_worker, nbatches, cfg: SamplerCfg | None = None):
        cfg = cfg or SamplerCfg()
        l = cfg.batch_size
        seeds = np.zeros(max(nbatches * l, 1), dtype=np.uint64)
        lens = np.zeros(max(nbatches * l, 1), dtype=np.uint32)
        counts = np.zeros(max(nbatches, 1), dtype=np.uint32)
        stats = np.zeros(8, dtype=np.uint64)
        self._chk(self.L.hsaw_gpu_encode_batches(self.h, C.byref(cfg), first_worker, nbatches,
                                                 _p(seeds, u64p), _p(lens, u32p), _p(counts, u32p),
                                                 _p(stats, u64p)))
        return (seeds[: nbatches * l].reshape(nbatches, l), lens[: nbatches * l].reshape(nbatches, l),
                counts[:nbatches], dict(zip(STAT_NAMES, (int(x) for x in stats))))

    def encode_stats(self, first_worker, nbatches, cfg: SamplerCfg | None = None) -> dict:
        """Work counters (attempts, draws, picks, algorithmic bytes, ...) of a batch range."""
        cfg = cfg or SamplerCfg()
        stats = np.zeros(8, dtype=np.uint64)
        self._chk(self.L.hsaw_gpu_encode_stats(self.h, C.byref(cfg), first_worker, nbatches,
                                               _p(stats, u64p)))
        return dict(zip(STAT_NAMES, (int(x) for x in stats)))

    def decode_walks(self, seeds, lens):
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        lens = np.ascontiguousarray(lens, dtype=np.uint32)
        nw = seeds.size
        eo = np.zeros(nw + 1, dtype=np.uint64)
        np.cumsum(lens, out=eo[1:])
        total = int(eo[-1])
        nodes = np.zeros(max(total + nw, 1), dtype=np.uint32)
        edges = np.zeros(max(total, 1), dtype=np.uint32)
        status = np.zeros(max(nw, 1), dtype=np.uint8)
        self._chk(self.L.hsaw_gpu_decode_walks(self.h, nw, _p(seeds, u64p), _p(lens, u32p),
                                               _p(eo, u64p), _p(nodes, u32p), _p(edges, u32p),
                                               _p(status, u8p)))
        return eo, nodes[: total + nw], edges[:total], status[:nw]

    def stream(self, seed=0, cfg: SamplerCfg | None = None) -> "Stream":
        return Stream(self, seed, cfg or SamplerCfg())

    def walkset(self, limit, set_off, items) -> "WalkSet":
        return WalkSet(self, limit, set_off, items)

    def rr_node_sets(self, state: int, count: int):
        """hsaw_gpu_rr_node_sets -> (WalkSet over node ids, state_after)."""
        s, h, total = C.c_uint64(state), C.c_void_p(), C.c_uint64()
        self._chk(self.L.hsaw_gpu_rr_node_sets(self.h, C.byref(s), count, C.byref(h),
                                               C.byref(total)))
        return WalkSet.adopt(self, h, count, total.value), s.value

    # ---- greedy / coverage
    def greedy(self, k, *, stream=None, walkset=None, kind=KIND_EDGE, off=0, cnt=None, cand=None):
        src = stream if stream is not None else walkset
        cnt = src.count - off if cnt is None else cnt
        ca = None if cand is None else np.ascontiguousarray(cand, dtype=np.uint32)
        if ca is not None and ca.size == 0:
            ca_ptr, nc = C.cast(C.c_void_p(1), u32p), 0  # explicit empty candidate set
        else:
            ca_ptr, nc = _p(ca, u32p), 0 if ca is None else ca.size
        sol = np.zeros(max(k, 1), dtype=np.uint32)
        cov = C.c_uint64()
        self._chk(self.L.hsaw_gpu_greedy(self.h, stream.h if stream is not None else None,
                                         walkset.h if walkset is not None else None, kind, off,
                                         cnt, ca_ptr, nc, k, _p(sol, u32p), C.byref(cov)))
        return sol[:k].copy(), cov.value

    def coverage_of(self, items, *, stream=None, walkset=None, kind=KIND_EDGE, off=0, cnt=None,
                    cand=None):
        src = stream if stream is not None else walkset
        cnt = src.count - off if cnt is None else cnt
        ca = None if cand is None else np.ascontiguousarray(cand, dtype=np.uint32)
        it = np.ascontiguousarray(items, dtype=np.uint32)
        cov = C.c_uint64()
        self._chk(self.L.hsaw_gpu_coverage_of(self.h, stream.h if stream is not None else None,
                                              walkset.h if walkset is not None else None, kind,
                                              off, cnt, _p(ca, u32p), 0 if ca is None else ca.size,
                                              _p(it, u32p) if it.size else None, it.size,
                                              C.byref(cov)))
        return cov.value


    def coverage_upper_bound(self, k, *, stream=None, walkset=None, kind=KIND_EDGE, off=0,
                             cnt=None, cand=None):
        """Upper bound of coverage_of over every set of <= k candidates (sum of the k largest
        per-item occurrence counts)."""
        src = stream if stream is not None else walkset
        cnt = src.count - off if cnt is None else cnt
        ca = None if cand is None else np.ascontiguousarray(cand, dtype=np.uint32)
        ub = C.c_uint64()
        self._chk(self.L.hsaw_gpu_coverage_upper_bound(
            self.h, stream.h if stream is not None else None,
            walkset.h if walkset is not None else None, kind, off, cnt, _p(ca, u32p),
            0 if ca is None else ca.size, k, C.byref(ub)))
        return ub.value


class Stream:
    """hsaw_gpu_stream == SampleStream (proj/include/hsaw/sampler.hpp:133-163)."""

    def __init__(self, ctx: Context, seed: int, cfg: SamplerCfg):
        self.ctx, self.L, self.cfg, self.seed = ctx, ctx.L, cfg, seed
        self.h = C.c_void_p()
        ctx._chk(self.L.hsaw_gpu_stream_create(ctx.h, seed, C.byref(cfg), C.byref(self.h)))

    def close(self):
        if self.h:
            self.L.hsaw_gpu_stream_destroy(self.h)
            self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def keep(self, nodes=True, edges=True):
        """hsaw_gpu_stream_keep: which item arrays the pool holds (before sampling)."""
        self.ctx._chk(self.L.hsaw_gpu_stream_keep(self.h, int(nodes), int(edges)))
        return self

    def restrict(self, domain, allowed):
        """hsaw_gpu_stream_restrict: start domain + allowed byte mask (partitioned sampling)."""
        d = np.ascontiguousarray(domain, dtype=np.uint32)
        a = np.ascontiguousarray(allowed, dtype=np.uint8)
        self.ctx._chk(self.L.hsaw_gpu_stream_restrict(self.h, _p(d, u32p), d.size,
                                                      a.ctypes.data_as(C.POINTER(C.c_uint8))))
        return self

    def crossings(self, min_accepted) -> int:
        c = C.c_uint64()
        self.ctx._chk(self.L.hsaw_gpu_stream_crossings(self.h, min_accepted, C.byref(c)))
        return c.value

    def ensure(self, min_accepted):
        self.ctx._chk(self.L.hsaw_gpu_stream_ensure(self.h, min_accepted))

    def sample_range(self, first_batch, nbatches) -> int:
        acc = C.c_uint64()
        self.ctx._chk(self.L.hsaw_gpu_stream_sample_range(self.h, first_batch, nbatches,
                                                          C.byref(acc)))
        return acc.value

    def size(self):
        a, b, e = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.ctx._chk(self.L.hsaw_gpu_stream_size(self.h, C.byref(a), C.byref(b), C.byref(e)))
        return a.value, b.value, e.value

    @property
    def count(self) -> int:
        return self.size()[0]

    def counters_for(self, min_accepted):
        at, ac = C.c_uint64(), C.c_uint64()
        self.ctx._chk(self.L.hsaw_gpu_stream_counters(self.h, min_accepted, C.byref(at),
                                                      C.byref(ac)))
        return at.value, ac.value

    def local_cut(self, min_local):
        nb, ac = C.c_uint64(), C.c_uint64()
        self.ctx._chk(self.L.hsaw_gpu_stream_local_cut(self.h, min_local, C.byref(nb),
                                                       C.byref(ac)))
        return nb.value, ac.value

    def collect_stats(self, on: bool = True):
        self.ctx._chk(self.L.hsaw_gpu_stream_collect_stats(self.h, int(on)))

    def stats(self) -> dict:
        st = np.zeros(8, dtype=np.uint64)
        self.ctx._chk(self.L.hsaw_gpu_stream_stats(self.h, _p(st, u64p)))
        return dict(zip(STAT_NAMES, (int(x) for x in st)))

    def export(self, off=0, cnt=None, attempts=0, nodes=True, edges=True) -> Pool:
        """Host copy of walks [off, off + cnt). nodes / edges False: skip that array (a stream
        that keeps only one kind, see keep())."""
        want_nodes, want_edges = nodes, edges
        cnt = self.count - off if cnt is None else cnt
        te = C.c_uint64()
        self.ctx._chk(self.L.hsaw_gpu_stream_slice_edges(self.h, off, cnt, C.byref(te)))
        te = te.value
        eo = np.zeros(cnt + 1, dtype=np.uint64)
        nodes = np.zeros(max(te + cnt, 1), dtype=np.uint32)
        edges = np.zeros(max(te, 1), dtype=np.uint32)
        tw = np.zeros(max(cnt, 1), dtype=np.uint64)
        ts = np.zeros(max(cnt, 1), dtype=np.uint32)
        self.ctx._chk(self.L.hsaw_gpu_stream_export(self.h, off, cnt, _p(eo, u64p),
                                                    _p(nodes, u32p) if want_nodes else None,
                                                    _p(edges, u32p) if want_edges else None,
                                                    _p(tw, u64p), _p(ts, u32p)))
        return Pool(attempts, eo, nodes[: te + cnt], edges[:te], tw[:cnt], ts[:cnt])

    def to_pool(self, min_accepted) -> Pool:
        """SampleStream::to_pool (proj/src/sampler.cpp:484-493)."""
        attempts, accepted = self.counters_for(min_accepted)
        return self.export(0, accepted, attempts)


class WalkSet:
    """hsaw_gpu_walkset: raw item sets for the fixed-walk-set parity mode."""

    def __init__(self, ctx: Context, limit, set_off, items):
        self.ctx, self.L = ctx, ctx.L
        set_off = np.ascontiguousarray(set_off, dtype=np.uint64)
        items = np.ascontiguousarray(items, dtype=np.uint32)
        self.count = set_off.size - 1
        self.h = C.c_void_p()
        ctx._chk(self.L.hsaw_gpu_walkset_import(ctx.h, limit, self.count, _p(set_off, u64p),
                                                _p(items, u32p) if items.size else None,
                                                C.byref(self.h)))

    @classmethod
    def adopt(cls, ctx, handle, count, nitems) -> "WalkSet":
        self = cls.__new__(cls)
        self.ctx, self.L, self.h, self.count, self.nitems = ctx, ctx.L, handle, count, nitems
        return self

    def export(self):
        """(set_off u64[count + 1], items) host copies."""
        off = np.zeros(self.count + 1, dtype=np.uint64)
        self.ctx._chk(self.L.hsaw_gpu_walkset_export(self.h, _p(off, u64p), None))
        items = np.zeros(max(int(off[-1]), 1), dtype=np.uint32)
        self.ctx._chk(self.L.hsaw_gpu_walkset_export(self.h, None, _p(items, u32p)))
        return off, items[: int(off[-1])]

    def close(self):
        if self.h:
            self.L.hsaw_gpu_walkset_destroy(self.h)
            self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class Rounds:
    """hsaw_gpu_rounds: greedy max-cover split into host-visible steps (sharded solves).
    d_counts / list buffers are raw DEVICE pointers owned by the caller (e.g. torch tensors)."""

    def __init__(self, ctx: Context, d_counts_ptr: int, *, stream=None, walkset=None,
                 kind=KIND_EDGE, off=0, cnt=0, cand=None):
        self.ctx, self.L = ctx, ctx.L
        ca = None if cand is None else np.ascontiguousarray(cand, dtype=np.uint32)
        if ca is not None and ca.size == 0:
            ca_ptr, nc = C.cast(C.c_void_p(1), u32p), 0
        else:
            ca_ptr, nc = _p(ca, u32p), 0 if ca is None else ca.size
        self.h = C.c_void_p()
        ctx._chk(self.L.hsaw_gpu_rounds_begin(ctx.h, stream.h if stream is not None else None,
                                              walkset.h if walkset is not None else None, kind,
                                              off, cnt, ca_ptr, nc, C.c_void_p(d_counts_ptr),
                                              C.byref(self.h)))
        self.occurrences = int(self.L.hsaw_gpu_rounds_occurrences(self.h))

    def select(self):
        item, gain = C.c_uint32(), C.c_uint64()
        self.ctx._chk(self.L.hsaw_gpu_rounds_select(self.h, C.byref(item), C.byref(gain)))
        return item.value, gain.value

    def cover(self, item: int, d_list_ptr: int, list_cap: int) -> int:
        n = C.c_uint64()
        self.ctx._chk(self.L.hsaw_gpu_rounds_cover(self.h, item, C.c_void_p(d_list_ptr), list_cap,
                                                   C.byref(n)))
        return n.value

    def apply(self, d_items_ptr: int, n: int):
        self.ctx._chk(self.L.hsaw_gpu_rounds_apply(self.h, C.c_void_p(d_items_ptr), n))

    def close(self):
        if self.h:
            self.L.hsaw_gpu_rounds_end(self.h)
            self.h = C.c_void_p()

"""ctypes binding of include/hsaw_host.h — the C view of the C++ host layer (hsaw_b200.hpp).

Plumbing for tests/ and bench.py. Loaders, schedule and the stopping rule run on the CPU (they are
host code in the reference too); everything that samples or runs greedy needs the CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _build
from .capi import HsawError, _p, f64p, u32p, u64p

WEIGHT_GIVEN, WEIGHT_INDEGREE, WEIGHT_RANDOM = 0, 1, 2


class Result(C.Structure):
    _fields_ = [("k", C.c_uint32), ("iterations", C.c_uint32), ("coverage", C.c_uint64),
                ("samples_used", C.c_uint64), ("attempts", C.c_uint64),
                ("est_suspension", C.c_double), ("wall_time_s", C.c_double),
                ("sample_s", C.c_double), ("greedy_s", C.c_double), ("check_s", C.c_double),
                ("passed_check", C.c_int32)]


_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(_build.HOST_SO):
        raise ImportError(f"{_build.HOST_SO} is missing: run __graft_entry__.build()")
    C.CDLL(_build.GPU_SO, mode=C.RTLD_GLOBAL)
    L = C.CDLL(_build.HOST_SO)
    vp, vpp = C.c_void_p, C.POINTER(C.c_void_p)
    L.hsawh_last_error.restype = C.c_char_p
    L.hsawh_graph_load_edge_list.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.c_int, C.c_char_p, vpp]
    L.hsawh_graph_build.argtypes = [C.c_uint32, C.c_uint64, u32p, u32p, f64p, C.c_int, C.c_uint64, vpp]
    L.hsawh_graph_build_device.argtypes = [C.c_uint32, C.c_uint64, u32p, u32p, f64p, C.c_int,
                                           C.c_int, vpp]
    L.hsawh_graph_synth.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, vpp]
    L.hsawh_graph_rmat.argtypes = [C.c_uint32, C.c_double, C.c_uint64, vpp]
    L.hsawh_graph_from_csr.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f64p, vpp]
    L.hsawh_graph_rmat_n.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, vpp]
    L.hsawh_graph_rmat_device.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.c_int, C.c_int, vpp]
    L.hsawh_graph_shell.argtypes = [C.c_uint32, C.c_uint32, vpp]
    L.hsawh_graph_ptrs.argtypes = [vp, C.POINTER(u64p), C.POINTER(u32p), C.POINTER(f64p)]
    L.hsawh_graph_ptrs.restype = None
    L.hsawh_suspects_random_n.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, f64p]
    L.hsawh_device_from_rmat.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, f64p, C.c_int, vp,
                                         C.c_int, vpp, vpp]
    L.hsawh_graph_save_cache.argtypes = [vp, C.c_char_p]
    L.hsawh_graph_load_cache.argtypes = [C.c_char_p, vpp]
    L.hsawh_graph_save_edge_list.argtypes = [vp, C.c_char_p]
    L.hsawh_graph_validate.argtypes = [vp]
    L.hsawh_graph_dims.argtypes = [vp, u32p, u32p]
    L.hsawh_graph_dims.restype = None
    L.hsawh_graph_copy.argtypes = [vp, u64p, u32p, f64p, f64p, u32p]
    L.hsawh_graph_copy.restype = None
    L.hsawh_graph_free.argtypes = [vp]
    L.hsawh_graph_free.restype = None
    L.hsawh_suspects_random.argtypes = [vp, C.c_uint32, C.c_uint64, f64p]
    L.hsawh_suspects_load.argtypes = [C.c_char_p, vp, f64p]
    L.hsawh_schedule.argtypes = [C.c_uint64, C.c_uint32, C.c_double, C.c_double, f64p, u32p]
    L.hsawh_check.argtypes = [C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_uint32,
                              C.c_double, C.c_double, C.c_uint32, C.POINTER(C.c_int), f64p]
    L.hsawh_device_create.argtypes = [vp, f64p, C.c_int, vp, vpp]
    L.hsawh_suspects_create.argtypes = [vp, f64p, vpp]
    L.hsawh_suspects_free.argtypes = [vp]
    L.hsawh_suspects_free.restype = None
    L.hsawh_device_create_vi.argtypes = [vp, vp, C.c_int, vp, vpp]
    L.hsawh_device_free.argtypes = [vp]
    L.hsawh_device_free.restype = None
    L.hsawh_device_ctx.argtypes = [vp]
    L.hsawh_device_ctx.restype = vp
    L.hsawh_interdict.argtypes = [vp, vp, f64p, C.c_int, u32p, C.c_uint64, C.c_uint32, C.c_double,
                                  C.c_double, C.c_uint64, C.c_uint32, C.c_uint64, C.c_int,
                                  C.POINTER(Result), u32p, C.c_char_p, C.c_uint64]
    L.hsawh_interdict_rng.argtypes = [vp, vp, f64p, C.c_int, u32p, C.c_uint64, C.c_uint32, C.c_double,
                                      C.c_double, C.c_uint64, C.c_uint32, C.c_uint64, C.c_int,
                                      C.c_int, C.POINTER(Result), u32p, C.c_char_p, C.c_uint64]
    L.hsawh_interdict_devices.argtypes = [vp, f64p, C.c_int, u32p, C.c_uint64, C.c_uint32, C.c_double,
                                          C.c_double, C.c_uint64, C.c_uint64, C.POINTER(C.c_int),
                                          C.c_uint32, C.POINTER(Result), u32p]
    L.hsawh_multi_transport.argtypes = [C.POINTER(C.c_int), C.c_uint32, C.c_char_p, C.c_uint64]
    L.hsawh_multi_transport.restype = None
    L.hsawh_sample.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_uint64, u64p, u64p]
    L.hsawh_graph_load_edge_list_device.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.c_int,
                                                    C.c_char_p, C.c_int, vpp]
    L.hsawh_graph_load_cache_device.argtypes = [C.c_char_p, C.c_int, vpp]
    L.hsawh_device_from_cache.argtypes = [C.c_char_p, C.c_int, vp, vpp]
    L.hsawh_device_from_edge_list.argtypes = [C.c_char_p, C.c_int, C.c_int, vp, vpp]
    L.hsawh_device_set_suspects.argtypes = [vp, vp, f64p]
    L.hsawh_lt_forward_simulate.argtypes = [vp, vp, f64p, u64p, u32p]
    L.hsawh_estimate_suspension.argtypes = [vp, vp, f64p, C.c_int, u32p, C.c_uint64, C.c_double,
                                            C.c_double, u64p, f64p, C.POINTER(C.c_int), u64p]
    L.hsawh_stream_samples.argtypes = [vp, f64p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, vpp]
    L.hsawh_pool_stats.argtypes = [vp, u64p, u64p, u64p]
    L.hsawh_pool_stats.restype = None
    L.hsawh_pool_copy.argtypes = [vp, u64p, u32p, u32p, u64p, u32p]
    L.hsawh_pool_copy.restype = None
    L.hsawh_pool_free.argtypes = [vp]
    L.hsawh_pool_free.restype = None
    L.hsawh_run_cli.argtypes = [C.c_int, C.POINTER(C.c_char_p)]
    u8p = C.POINTER(C.c_uint8)
    L.hsawh_partition.argtypes = [vp, C.c_uint32, C.c_int, C.c_uint64, C.c_char_p, C.c_uint32, u32p,
                                  u8p]
    L.hsawh_distributed_sample.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint32, u32p, u8p,
                                           C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, vpp,
                                           u64p, u64p, f64p, u64p]
    L.hsawh_baseline.argtypes = [vp, vp, f64p, C.c_int, C.c_int, C.c_uint32, u64p, C.c_uint32, u32p]
    L.hsawh_rr_node_sets.argtypes = [vp, u64p, C.c_uint32, u64p, u32p, C.c_uint64, u64p]
    L.hsawh_json_number.argtypes = [C.c_double, C.c_char_p, C.c_uint64]
    L.hsawh_json_number.restype = None
    _LIB = L
    return L


def _chk(rc):
    if rc:
        raise HsawError(rc, lib().hsawh_last_error().decode())


class Graph:
    """hsaw::ProbGraph handle."""

    def __init__(self, handle):
        self.h = handle
        n, m = C.c_uint32(), C.c_uint32()
        lib().hsawh_graph_dims(self.h, C.byref(n), C.byref(m))
        self.n, self.m = n.value, m.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().hsawh_graph_free(self.h)
            self.h = None

    @staticmethod
    def _new(fn, *args) -> "Graph":
        h = C.c_void_p()
        _chk(fn(*args, C.byref(h)))
        return Graph(h)

    @classmethod
    def load_edge_list(cls, path, mode=WEIGHT_INDEGREE, seed=0, symmetrize=False, mapping_out=None):
        return cls._new(lib().hsawh_graph_load_edge_list, str(path).encode(), mode, seed,
                        int(symmetrize), mapping_out.encode() if mapping_out else None)

    @classmethod
    def build(cls, n, u, v, w=None, mode=WEIGHT_INDEGREE, seed=0):
        u = np.ascontiguousarray(u, dtype=np.uint32)
        v = np.ascontiguousarray(v, dtype=np.uint32)
        wa = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
        return cls._new(lib().hsawh_graph_build, n, u.size, _p(u, u32p), _p(v, u32p),
                        _p(wa, f64p), mode, seed)

    @classmethod
    def build_device(cls, n, u, v, w=None, mode=WEIGHT_INDEGREE, device=0):
        """hsaw::build_graph_device: same ProbGraph as build(), sorted and summed on the GPU."""
        u = np.ascontiguousarray(u, dtype=np.uint32)
        v = np.ascontiguousarray(v, dtype=np.uint32)
        wa = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
        return cls._new(lib().hsawh_graph_build_device, n, u.size, _p(u, u32p), _p(v, u32p),
                        _p(wa, f64p), mode, device)

    @classmethod
    def synth(cls, n, density, seed):
        return cls._new(lib().hsawh_graph_synth, n, density, seed)

    @classmethod
    def rmat(cls, scale, edge_factor, seed=1):
        return cls._new(lib().hsawh_graph_rmat, scale, float(edge_factor), seed)

    @classmethod
    def rmat_n(cls, n, raw_edges, seed=1):
        """hsaw::rmat_graph_n on the host (sequential stream + std::sort; small shapes only)."""
        return cls._new(lib().hsawh_graph_rmat_n, n, raw_edges, seed)

    @classmethod
    def rmat_device(cls, n, raw_edges, seed=1, device=0, lean=False):
        """hsaw::rmat_graph_device: the same ProbGraph generated / sorted / summed on the GPU."""
        return cls._new(lib().hsawh_graph_rmat_device, n, raw_edges, seed, device, int(lean))

    @classmethod
    def shell(cls, n, m):
        """A ProbGraph carrying only n and m (the graph itself lives on the device)."""
        return cls._new(lib().hsawh_graph_shell, n, m)

    def views(self):
        """(in_offsets, in_src, in_cum) as zero-copy views of the ProbGraph's own vectors — valid
        while this Graph is alive."""
        o, s_, c = u64p(), u32p(), f64p()
        lib().hsawh_graph_ptrs(self.h, C.byref(o), C.byref(s_), C.byref(c))
        if self.m == 0:
            return (np.ctypeslib.as_array(o, shape=(self.n + 1,)), np.zeros(0, dtype=np.uint32),
                    np.zeros(0, dtype=np.float64))
        return (np.ctypeslib.as_array(o, shape=(self.n + 1,)),
                np.ctypeslib.as_array(s_, shape=(self.m,)),
                np.ctypeslib.as_array(c, shape=(self.m,)))

    @classmethod
    def from_csr(cls, n, m, in_offsets, in_src, in_cum):
        o = np.ascontiguousarray(in_offsets, dtype=np.uint64)
        s = np.ascontiguousarray(in_src, dtype=np.uint32)
        c = np.ascontiguousarray(in_cum, dtype=np.float64)
        return cls._new(lib().hsawh_graph_from_csr, n, m, _p(o, u64p), _p(s, u32p), _p(c, f64p))

    @classmethod
    def load_cache(cls, path):
        return cls._new(lib().hsawh_graph_load_cache, str(path).encode())

    @classmethod
    def load_edge_list_device(cls, path, mode=1, seed=0, symmetrize=False, mapping_out=None,
                              device=0):
        """hsaw::load_edge_list_device: text parse, id remap and build_graph on the GPU."""
        return cls._new(lib().hsawh_graph_load_edge_list_device, str(path).encode(), mode, seed,
                        int(symmetrize), str(mapping_out).encode() if mapping_out else None, device)

    @classmethod
    def load_cache_device(cls, path, device=0):
        """hsaw::load_cache_device: load_cache with decode / sums / validate() on the GPU."""
        return cls._new(lib().hsawh_graph_load_cache_device, str(path).encode(), device)

    def save_cache(self, path):
        _chk(lib().hsawh_graph_save_cache(self.h, str(path).encode()))

    def save_edge_list(self, path):
        _chk(lib().hsawh_graph_save_edge_list(self.h, str(path).encode()))

    def validate(self):
        _chk(lib().hsawh_graph_validate(self.h))

    def arrays(self):
        """(in_offsets, in_src, in_cum, weight, edge_dst) copies."""
        off = np.zeros(self.n + 1, dtype=np.uint64)
        src = np.zeros(max(self.m, 1), dtype=np.uint32)
        cum = np.zeros(max(self.m, 1), dtype=np.float64)
        w = np.zeros(max(self.m, 1), dtype=np.float64)
        dst = np.zeros(max(self.m, 1), dtype=np.uint32)
        lib().hsawh_graph_copy(self.h, _p(off, u64p), _p(src, u32p), _p(cum, f64p), _p(w, f64p),
                               _p(dst, u32p))
        m = self.m
        return off, src[:m], cum[:m], w[:m], dst[:m]

    def random_suspects(self, count, seed) -> np.ndarray:
        p = np.zeros(max(self.n, 1), dtype=np.float64)
        _chk(lib().hsawh_suspects_random(self.h, count, seed, _p(p, f64p)))
        return p[: self.n]

    def load_suspects(self, path) -> np.ndarray:
        p = np.zeros(max(self.n, 1), dtype=np.float64)
        _chk(lib().hsawh_suspects_load(str(path).encode(), self.h, _p(p, f64p)))
        return p[: self.n]


def random_suspects_n(n, count, seed) -> np.ndarray:
    """hsaw::random_suspects by node count (the draws do not depend on the edges)."""
    p = np.zeros(max(n, 1), dtype=np.float64)
    _chk(lib().hsawh_suspects_random_n(n, count, seed, _p(p, f64p)))
    return p[:n]


def schedule(M, k, eps, delta) -> dict:
    out = np.zeros(4, dtype=np.float64)
    t = C.c_uint32()
    _chk(lib().hsawh_schedule(M, k, eps, delta, _p(out, f64p), C.byref(t)))
    return dict(n_max=float(out[0]), lambda_=float(out[1]), lambda1=float(out[2]), t_max=t.value,
                lambda_samples=int(out[3]))


def check(cov_r, cov_rp, n_rp, M, k, eps, delta, t):
    ok, e = C.c_int(), C.c_double()
    _chk(lib().hsawh_check(float(cov_r), float(cov_rp), float(n_rp), M, k, eps, delta, t,
                           C.byref(ok), C.byref(e)))
    return bool(ok.value), e.value


class Suspects:
    """hsaw::SuspectSet built once from a dense p_of array (0 = not a suspect): the object a C++
    caller hands to DeviceGraph(g, vi), so per-call uploads do not rebuild it."""

    def __init__(self, graph: Graph, p_of):
        self.p_of = np.ascontiguousarray(p_of, dtype=np.float64)
        self.h = C.c_void_p()
        _chk(lib().hsawh_suspects_create(graph.h, _p(self.p_of, f64p), C.byref(self.h)))

    def close(self):
        if self.h:
            lib().hsawh_suspects_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceGraph:
    """hsaw::DeviceGraph: the graph + suspects uploaded to one GPU."""

    def __init__(self, graph: Graph, p_of, device=0, cuda_stream: int | None = None):
        self.graph = graph
        self.h = C.c_void_p()
        stream = C.c_void_p(cuda_stream) if cuda_stream else None
        if isinstance(p_of, Suspects):
            self.p_of = p_of.p_of
            _chk(lib().hsawh_device_create_vi(graph.h, p_of.h, device, stream, C.byref(self.h)))
            return
        self.p_of = np.ascontiguousarray(p_of, dtype=np.float64)
        _chk(lib().hsawh_device_create(graph.h, _p(self.p_of, f64p), device, stream,
                                       C.byref(self.h)))

    @classmethod
    def from_cache(cls, path, device=0, cuda_stream: int | None = None) -> "DeviceGraph":
        """hsaw::DeviceGraph::from_cache: HSAW1 file -> resident graph, no host CSR, no suspects."""
        self = cls.__new__(cls)
        self.graph, self.p_of, self.h = None, None, C.c_void_p()
        _chk(lib().hsawh_device_from_cache(str(path).encode(), device,
                                           C.c_void_p(cuda_stream) if cuda_stream else None,
                                           C.byref(self.h)))
        return self

    @classmethod
    def from_edge_list(cls, path, mode=1, device=0, cuda_stream: int | None = None):
        """hsaw::DeviceGraph::from_edge_list: text file -> resident graph (None: host loader needed)."""
        self = cls.__new__(cls)
        self.graph, self.p_of, self.h = None, None, C.c_void_p()
        _chk(lib().hsawh_device_from_edge_list(str(path).encode(), mode, device,
                                               C.c_void_p(cuda_stream) if cuda_stream else None,
                                               C.byref(self.h)))
        return self if self.h else None

    @classmethod
    def from_rmat(cls, n, raw_edges, seed, p_of=None, device=0, cuda_stream: int | None = None,
                  want_host=False) -> "DeviceGraph":
        """hsaw::DeviceGraph::from_rmat: R-MAT graph generated on the device and installed where it
        lies. self.graph is the lean host copy (want_host) or a shell with n and m only."""
        self = cls.__new__(cls)
        self.p_of = None if p_of is None else np.ascontiguousarray(p_of, dtype=np.float64)
        self.h, gh = C.c_void_p(), C.c_void_p()
        _chk(lib().hsawh_device_from_rmat(n, raw_edges, seed, _p(self.p_of, f64p), device,
                                          C.c_void_p(cuda_stream) if cuda_stream else None,
                                          int(want_host), C.byref(self.h), C.byref(gh)))
        self.graph = Graph(gh)
        return self

    def set_suspects(self, graph: "Graph", p_of):
        self.graph = graph
        self.p_of = np.ascontiguousarray(p_of, dtype=np.float64)
        _chk(lib().hsawh_device_set_suspects(self.h, graph.h, _p(self.p_of, f64p)))

    def close(self):
        if self.h:
            lib().hsawh_device_free(self.h)
            self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def ctx_handle(self):
        return lib().hsawh_device_ctx(self.h)

    def stage_times(self, reset=False) -> dict:
        from . import capi
        ms = np.zeros(len(capi.STAGE_NAMES), dtype=np.float64)
        cnt = np.zeros(len(capi.STAGE_NAMES), dtype=np.uint64)
        rc = capi.lib().hsaw_gpu_stage_times(self.ctx_handle(), _p(ms, f64p), _p(cnt, u64p),
                                             int(reset))
        if rc:
            raise HsawError(rc, "stage_times")
        return {n: (float(ms[i]), int(cnt[i])) for i, n in enumerate(capi.STAGE_NAMES)}

    def launches(self) -> int:
        from . import capi
        return int(capi.lib().hsaw_gpu_launch_count(self.ctx_handle()))

    def sample(self, target, seed=0, max_attempts=100_000_000):
        """`hsaw sample` without the dump: (attempts, accepted) of the pool for `target`."""
        at, ac = C.c_uint64(), C.c_uint64()
        _chk(lib().hsawh_sample(self.h, target, seed, max_attempts, C.byref(at), C.byref(ac)))
        return at.value, ac.value


def interdict(graph: Graph, p_of, kind, k, eps, delta, seed=0, cand=None, batch_size=10,
              max_attempts=100_000_000, device=0, dg: DeviceGraph | None = None,
              want_json=False, rng_mode=0) -> dict:
    """esia (kind 0) / nsia (kind 1). With dg the graph is already on the device. rng_mode 1: the
    Philox per-walk throughput mode (statistical parity only)."""
    p = np.ascontiguousarray(p_of, dtype=np.float64)
    ca = None if cand is None else np.ascontiguousarray(cand, dtype=np.uint32)
    if ca is not None and ca.size == 0:
        ca_ptr, nc = C.cast(C.c_void_p(8), u32p), 0
    else:
        ca_ptr, nc = _p(ca, u32p), 0 if ca is None else ca.size
    res = Result()
    sol = np.zeros(max(k, 1), dtype=np.uint32)
    buf = C.create_string_buffer(1 << 16)
    _chk(lib().hsawh_interdict_rng(dg.h if dg is not None else None, graph.h, _p(p, f64p), kind,
                                   ca_ptr, nc, k, eps, delta, seed, batch_size, max_attempts,
                                   device, rng_mode, C.byref(res), _p(sol, u32p), buf, len(buf)))
    out = dict(kind="edge" if kind == 0 else "node", k=res.k, epsilon=eps, delta=delta,
               solution=[int(x) for x in sol[:k]], est_suspension=res.est_suspension,
               coverage=res.coverage, samples_used=res.samples_used, attempts=res.attempts,
               iterations=res.iterations, passed_check=bool(res.passed_check))
    if want_json:
        out["json"] = buf.value.decode()
        out["timing"] = dict(wall_time_s=res.wall_time_s, sample_s=res.sample_s,
                             greedy_s=res.greedy_s, check_s=res.check_s)
    return out


def multi_transport(devices) -> str:
    dev = (C.c_int * len(devices))(*devices)
    buf = C.create_string_buffer(128)
    lib().hsawh_multi_transport(dev, len(devices), buf, len(buf))
    return buf.value.decode()


def interdict_devices(graph: Graph, p_of, kind, k, eps, delta, devices, seed=0, cand=None,
                      max_attempts=100_000_000, with_timing=False) -> dict:
    """esia / nsia with InterdictionOptions::devices (the C++ multi-device solve, host/multi.cpp)."""
    p = np.ascontiguousarray(p_of, dtype=np.float64)
    ca = None if cand is None else np.ascontiguousarray(cand, dtype=np.uint32)
    dev = (C.c_int * len(devices))(*devices)
    res = Result()
    sol = np.zeros(max(k, 1), dtype=np.uint32)
    _chk(lib().hsawh_interdict_devices(graph.h, _p(p, f64p), kind, _p(ca, u32p),
                                       0 if ca is None else ca.size, k, eps, delta, seed,
                                       max_attempts, dev, len(devices), C.byref(res), _p(sol, u32p)))
    out = dict(kind="edge" if kind == 0 else "node", k=res.k, epsilon=eps, delta=delta,
               solution=[int(x) for x in sol[:k]], est_suspension=res.est_suspension,
               coverage=res.coverage, samples_used=res.samples_used, attempts=res.attempts,
               iterations=res.iterations, passed_check=bool(res.passed_check))
    if with_timing:  # (kept out of the default result: it is compared with golden results)
        out["timing"] = dict(wall_time_s=res.wall_time_s, sample_s=res.sample_s,
                             greedy_s=res.greedy_s, check_s=res.check_s)
    return out


def lt_forward_simulate(graph: Graph, p_of, state, dg: DeviceGraph | None = None):
    """hsaw::lt_forward_simulate(g, vi, s) -> (infected, state_after)."""
    p = np.ascontiguousarray(p_of, dtype=np.float64)
    s, out = C.c_uint64(state), C.c_uint32()
    _chk(lib().hsawh_lt_forward_simulate(dg.h if dg is not None else None, graph.h, _p(p, f64p),
                                         C.byref(s), C.byref(out)))
    return int(out.value), s.value


def estimate_suspension(graph: Graph, p_of, kind, ids, eps, delta, state,
                        dg: DeviceGraph | None = None) -> dict:
    """hsaw::estimate_suspension(g, vi, removal, eps, delta, s) -> dict(value, capped, runs, state)."""
    p = np.ascontiguousarray(p_of, dtype=np.float64)
    a = np.ascontiguousarray(ids, dtype=np.uint32)
    buf = a if a.size else np.zeros(1, dtype=np.uint32)
    s, v, cp, runs = C.c_uint64(state), C.c_double(), C.c_int(), C.c_uint64()
    _chk(lib().hsawh_estimate_suspension(dg.h if dg is not None else None, graph.h, _p(p, f64p),
                                         kind, _p(buf, u32p), a.size, eps, delta, C.byref(s),
                                         C.byref(v), C.byref(cp), C.byref(runs)))
    return dict(value=v.value, capped=bool(cp.value), runs=int(runs.value), state=s.value)


BASELINES = {"pagerank": 0, "maxdegree": 1, "randomized": 2, "infmax-v": 3, "infmax-vi": 4}


def baseline(graph: Graph, p_of, kind, mode, k, state, infmax_samples=100000,
             dg: "DeviceGraph | None" = None):
    """hsaw::baseline(...) -> (ids, state_after). mode 0 edge / 1 node."""
    p = np.ascontiguousarray(p_of, dtype=np.float64)
    ids = np.zeros(max(k, 1), dtype=np.uint32)
    s = C.c_uint64(state)
    _chk(lib().hsawh_baseline(dg.h if dg is not None else None, graph.h, _p(p, f64p),
                              BASELINES[kind], mode, k, C.byref(s), infmax_samples, _p(ids, u32p)))
    return [int(x) for x in ids[:k]], s.value


def rr_node_sets(dg: "DeviceGraph", state, count):
    """hsaw::rr_node_sets(dg, s, count) -> (set_off, items, state_after)."""
    off = np.zeros(count + 1, dtype=np.uint64)
    cap = max(4096, count * 64)
    while True:
        items = np.zeros(cap, dtype=np.uint32)
        s, total = C.c_uint64(state), C.c_uint64()
        _chk(lib().hsawh_rr_node_sets(dg.h, C.byref(s), count, _p(off, u64p), _p(items, u32p), cap,
                                      C.byref(total)))
        if total.value <= cap:
            return off, items[: total.value].copy(), s.value
        cap = total.value


PART_METHODS = {"hash": 0, "labelprop": 1, "external": 2}


def partition(graph: Graph, p, method="hash", seed=0, part_file=None, hops=0):
    """hsaw::partition_graph + extend_partition(hops) -> (assign u32[n], extended u8[p, n])."""
    assign = np.zeros(max(graph.n, 1), dtype=np.uint32)
    ext = np.zeros((p, graph.n), dtype=np.uint8)
    _chk(lib().hsawh_partition(graph.h, p, PART_METHODS[method], seed,
                               str(part_file).encode() if part_file else None, hops,
                               _p(assign, u32p), ext.ctypes.data_as(C.POINTER(C.c_uint8))))
    return assign[: graph.n], ext


def distributed_sample(dg: "DeviceGraph", assign, extended, total_target, seed=0, hops=0,
                       batch_size=10, max_attempts=100_000_000) -> dict:
    """hsaw::distributed_sample(dg, part, total_target, seed, cfg) -> dict(pool, crossings,
    attempts, crossing_fraction, targets)."""
    a = np.ascontiguousarray(assign, dtype=np.uint32)
    e = np.ascontiguousarray(extended, dtype=np.uint8)
    p = e.shape[0]
    h, cr, at, fr = C.c_void_p(), C.c_uint64(), C.c_uint64(), C.c_double()
    tg = np.zeros(p, dtype=np.uint64)
    _chk(lib().hsawh_distributed_sample(dg.h, a.size, p, hops, _p(a, u32p),
                                        e.ctypes.data_as(C.POINTER(C.c_uint8)), total_target, seed,
                                        batch_size, max_attempts, C.byref(h), C.byref(cr),
                                        C.byref(at), C.byref(fr), _p(tg, u64p)))
    try:
        pool = _pool_from_handle(h)
    finally:
        lib().hsawh_pool_free(h)
    return dict(pool=pool, crossings=cr.value, attempts=at.value, crossing_fraction=fr.value,
                targets=[int(x) for x in tg])


def _pool_from_handle(h):
    from .capi import Pool
    ns, at, te = C.c_uint64(), C.c_uint64(), C.c_uint64()
    lib().hsawh_pool_stats(h, C.byref(ns), C.byref(at), C.byref(te))
    ns, at, te = ns.value, at.value, te.value
    eo = np.zeros(ns + 1, dtype=np.uint64)
    nodes = np.zeros(max(te + ns, 1), dtype=np.uint32)
    edges = np.zeros(max(te, 1), dtype=np.uint32)
    tw = np.zeros(max(ns, 1), dtype=np.uint64)
    ts = np.zeros(max(ns, 1), dtype=np.uint32)
    lib().hsawh_pool_copy(h, _p(eo, u64p), _p(nodes, u32p), _p(edges, u32p), _p(tw, u64p),
                          _p(ts, u32p))
    return Pool(at, eo, nodes[: te + ns], edges[:te], tw[:ns], ts[:ns])


def stream_samples(graph: Graph, p_of, target, seed=0, batch_size=10, max_attempts=100_000_000):
    """Reference-signature stream_samples(g, vi, workers, target, seed, cfg) -> host pool."""
    from .capi import Pool
    p = np.ascontiguousarray(p_of, dtype=np.float64)
    h = C.c_void_p()
    _chk(lib().hsawh_stream_samples(graph.h, _p(p, f64p), target, seed, batch_size, max_attempts,
                                    C.byref(h)))
    try:
        ns, at, te = C.c_uint64(), C.c_uint64(), C.c_uint64()
        lib().hsawh_pool_stats(h, C.byref(ns), C.byref(at), C.byref(te))
        ns, at, te = ns.value, at.value, te.value
        eo = np.zeros(ns + 1, dtype=np.uint64)
        nodes = np.zeros(max(te + ns, 1), dtype=np.uint32)
        edges = np.zeros(max(te, 1), dtype=np.uint32)
        tw = np.zeros(max(ns, 1), dtype=np.uint64)
        ts = np.zeros(max(ns, 1), dtype=np.uint32)
        lib().hsawh_pool_copy(h, _p(eo, u64p), _p(nodes, u32p), _p(edges, u32p), _p(tw, u64p),
                              _p(ts, u32p))
        return Pool(at, eo, nodes[: te + ns], edges[:te], tw[:ns], ts[:ns])
    finally:
        lib().hsawh_pool_free(h)


def json_number(x: float) -> str:
    buf = C.create_string_buffer(64)
    lib().hsawh_json_number(float(x), buf, len(buf))
    return buf.value.decode()


def run_cli(args: list[str]) -> int:
    arr = (C.c_char_p * len(args))(*[a.encode() for a in args])
    return lib().hsawh_run_cli(len(args), arr)

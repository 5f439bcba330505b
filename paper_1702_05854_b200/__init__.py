"""B200-native HSAW sampling + greedy max-cover (the eSIA/nSIA hot path of arXiv 1702.05854).

The product is two native libraries built in-tree by `_build.py`:
  lib/libhsaw_gpu.so   hand-written sm_100a CUDA kernels behind the C-ABI of include/hsaw_gpu.h
  lib/libhsaw_host.so  C++ host layer with the reference's own `hsaw::` entry points (esia, nsia,
                       stream_samples, loaders, CLI) on top of that C-ABI
`capi` / `hostapi` are thin ctypes bindings used by tests/ and bench.py. Nothing in this package
imports oracle/, and nothing falls back to a CPU path.
"""
from . import _build  # noqa: F401

__all__ = ["_build"]

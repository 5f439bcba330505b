#!/bin/bash
# compute-sanitizer over the kernels added in round 2 (dense greedy instance, window histogram,
# flat coverage, Floyd tortoise, regenerated in_cum, side-stream replay)
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_greedy.py -x -q -m gpu -k "micro or golden or random_instances or empty or stream_greedy or upper_bound or monotone" > gpurun_out/r02e_sanitizer_memcheck_greedy.txt 2>&1; echo "memcheck greedy rc=$?"; tail -4 gpurun_out/r02e_sanitizer_memcheck_greedy.txt
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_sampler.py -x -q -m gpu -k "floyd or regenerates or long_walk or overflow" > gpurun_out/r02e_sanitizer_memcheck_sampler.txt 2>&1; echo "memcheck sampler rc=$?"; tail -4 gpurun_out/r02e_sanitizer_memcheck_sampler.txt
HSAW_HIST_FORCE_WINDOWS=1 timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_greedy.py -x -q -m gpu -k "partitioned_histogram and compact-plain" > gpurun_out/r02e_sanitizer_memcheck_windows.txt 2>&1; echo "memcheck windows rc=$?"; tail -4 gpurun_out/r02e_sanitizer_memcheck_windows.txt
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_greedy.py -x -q -m gpu -k "(micro or golden or stream_greedy or upper_bound) and (dense-fat or dense-compact-exact)" > gpurun_out/r02e_sanitizer_racecheck_greedy.txt 2>&1; echo "racecheck greedy rc=$?"; tail -4 gpurun_out/r02e_sanitizer_racecheck_greedy.txt

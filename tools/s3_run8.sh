#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_greedy.py -x -q -m gpu 2>&1 | tail -2
echo "== smem windows"; REPS=2 NO_TOUCH=1 python tools/esia_stages.py c4 2>&1 | tail -1
echo "== bits 8"; HSAW_HIST_BITS=8 REPS=2 NO_TOUCH=1 python tools/esia_stages.py c4 2>&1 | tail -1
HSAW_UPLOAD_TIMING=1 python bench.py --no-esia --no-cpu-baseline --no-philox --no-suspension --steps 3 2> gpurun_out/s3r8_bench.err > gpurun_out/s3r8_bench.json; grep "hsaw upload\|bench e2e" gpurun_out/s3r8_bench.err | tail -12

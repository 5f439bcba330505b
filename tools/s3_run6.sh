#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_greedy.py tests/test_gpu_fullsize.py tests/test_gpu_interdiction.py tests/test_gpu_sharded.py tests/test_gpu_baseline.py tests/test_gpu_sampler.py -x -q -m gpu > gpurun_out/s3r6_tests.log 2>&1; tail -4 gpurun_out/s3r6_tests.log
HSAW_UPLOAD_TIMING=1 python bench.py --no-esia --no-cpu-baseline --no-philox --no-suspension --steps 3 2> gpurun_out/s3r6_bench.err > gpurun_out/s3r6_bench.json; grep "hsaw upload" gpurun_out/s3r6_bench.err | tail -8; python -c "
import json; d=json.loads(open('gpurun_out/s3r6_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e'])"

#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sampler.py tests/test_gpu_greedy.py tests/test_gpu_fullsize.py tests/test_gpu_interdiction.py -x -q -m gpu > gpurun_out/s3r13_tests.log 2>&1; tail -4 gpurun_out/s3r13_tests.log
HSAW_UPLOAD_TIMING=1 python bench.py --no-cpu-baseline --no-philox --steps 5 2> gpurun_out/s3r13_bench.err > gpurun_out/s3r13_bench.json; grep "hsaw upload\|bench e2e" gpurun_out/s3r13_bench.err | tail -7; python -c "
import json; d=json.loads(open('gpurun_out/s3r13_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']); print(d['esia_k1000'])"
python bench.py --workload c2 --no-cpu-baseline --no-philox --steps 10 2>/dev/null > gpurun_out/s3r13_bench_c2.json; python -c "
import json; d=json.loads(open('gpurun_out/s3r13_bench_c2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']); print(d['esia'], d['esia_k1000'])"

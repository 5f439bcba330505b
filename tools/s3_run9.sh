#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/s3r9_tests.log 2>&1; tail -3 gpurun_out/s3r9_tests.log
HSAW_UPLOAD_TIMING=1 python bench.py --no-cpu-baseline --no-philox --steps 5 2> gpurun_out/s3r9_bench.err > gpurun_out/s3r9_bench.json; grep "hsaw upload\|bench e2e" gpurun_out/s3r9_bench.err | tail -7; python -c "
import json; d=json.loads(open('gpurun_out/s3r9_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']); print(d['esia_k1000']); print(d['suspension'])"

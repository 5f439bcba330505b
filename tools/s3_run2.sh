#!/bin/bash
# session 3, run 2: dense greedy parity, then C4 eSIA timing + upload phase timing
mkdir -p gpurun_out
python -m pytest tests/test_gpu_greedy.py -x -q -m gpu > gpurun_out/s3r2_greedy.log 2>&1; tail -5 gpurun_out/s3r2_greedy.log
python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_interdiction.py tests/test_gpu_sharded.py tests/test_gpu_baseline.py -x -q -m gpu > gpurun_out/s3r2_full.log 2>&1; tail -5 gpurun_out/s3r2_full.log
HSAW_UPLOAD_THREADS=8 HSAW_UPLOAD_TIMING=1 python bench.py --no-cpu-baseline --no-philox --no-suspension --steps 3 > gpurun_out/s3r2_bench_c4.json 2> gpurun_out/s3r2_bench_c4.err
grep "hsaw upload" gpurun_out/s3r2_bench_c4.err | tail -12
python - <<'PY'
import json
d=json.loads(open('gpurun_out/s3r2_bench_c4.json').read().strip().splitlines()[-1])
print('value',d['value'],'e2e',d['e2e']); print(d['esia_k1000'])
PY

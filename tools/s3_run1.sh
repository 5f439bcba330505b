#!/bin/bash
# session 3, run 1: Floyd + partition tests, default bench (e2e OOM fix), upload thread sweep
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sampler.py tests/test_gpu_partition.py tests/test_gpu_greedy.py -x -q -m gpu > gpurun_out/s3r1_tests.log 2>&1; tail -3 gpurun_out/s3r1_tests.log
python bench.py > gpurun_out/s3r1_bench_c4.json 2> gpurun_out/s3r1_bench_c4.err; tail -c 300 gpurun_out/s3r1_bench_c4.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/s3r1_bench_c4.json').read().strip().splitlines()[-1])
print('value',d['value'],'e2e',d['e2e']); print(d['esia_k1000'])
PY
for cfg in "4 4" "8 4" "12 4" "16 4" "8 16" "16 16"; do
  set -- $cfg
  HSAW_UPLOAD_THREADS=$1 HSAW_UPLOAD_CHUNK_MB=$2 python bench.py --no-esia --no-cpu-baseline --no-philox --no-suspension --steps 3 > gpurun_out/s3r1_up_$1_$2.json 2>/dev/null
  python - "$1" "$2" <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/s3r1_up_{sys.argv[1]}_{sys.argv[2]}.json').read().strip().splitlines()[-1])
print('threads',sys.argv[1],'chunkMB',sys.argv[2],'e2e',d['e2e']['value'],'ms/call',d['e2e']['ms_per_call'],d['e2e'].get('error'))
PY
done

#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sampler.py -x -q -m gpu -k "upload" 2>&1 | tail -2
for t in 8 12 16; do
echo "== check threads $t"
HSAW_UPLOAD_CHECK_THREADS=$t HSAW_UPLOAD_TIMING=1 python bench.py --no-esia --no-cpu-baseline --no-philox --no-suspension --steps 3 2> gpurun_out/s3r14_bench.err > gpurun_out/s3r14_bench.json; grep "hsaw upload\|bench e2e" gpurun_out/s3r14_bench.err | tail -6 | grep -v alloc; python -c "
import json; d=json.loads(open('gpurun_out/s3r14_bench.json').read().strip().splitlines()[-1]); print(d['e2e']['value'], d['e2e']['ms_per_call'])"
done
echo "== regen off"; HSAW_UPLOAD_REGEN=0 python bench.py --no-esia --no-cpu-baseline --no-philox --no-suspension --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['e2e']['value'], d['e2e']['ms_per_call'])"

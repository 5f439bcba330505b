#!/bin/bash
mkdir -p gpurun_out
for b in 8 12 16 20; do echo "== hist bits $b"; HSAW_HIST_BITS=$b REPS=2 NO_TOUCH=1 python tools/esia_stages.py c4 2>&1 | tail -1; done
HSAW_UPLOAD_TIMING=1 python bench.py --no-esia --no-cpu-baseline --no-philox --no-suspension --steps 3 2> gpurun_out/s3r7_bench.err > gpurun_out/s3r7_bench.json; grep "hsaw upload" gpurun_out/s3r7_bench.err | tail -5; python -c "
import json; d=json.loads(open('gpurun_out/s3r7_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e'])"

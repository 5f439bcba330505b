#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_sampler.py tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/s3r15_tests.log 2>&1; tail -3 gpurun_out/s3r15_tests.log
python bench.py --no-esia --no-cpu-baseline --no-philox --no-suspension --no-e2e --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['stage_ms'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"distinct_kernel<.*1024" -s 3 -c 1 -f -o gpurun_out/s3r15_c4_k2b python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-esia --no-philox > /dev/null 2> gpurun_out/s3r15_k2b.err
ncu -i gpurun_out/s3r15_c4_k2b.ncu-rep --page details --csv > gpurun_out/s3r15_c4_k2b_details.csv 2>/dev/null
python tools/ncu_key.py gpurun_out/s3r15_c4_k2b.ncu-rep
ncu -i gpurun_out/s3r15_c4_k2b.ncu-rep --page source --csv > gpurun_out/s3r15_c4_k2b_source.csv 2>/dev/null; wc -l gpurun_out/s3r15_c4_k2b_source.csv

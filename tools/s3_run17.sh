#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/s3r17_tests.log 2>&1; tail -3 gpurun_out/s3r17_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
(time python bench.py) > gpurun_out/s3r17_bench.json 2> gpurun_out/s3r17_bench.err; tail -4 gpurun_out/s3r17_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/s3r17_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']); print(d['roofline']['frac'], d['roofline']['traffic'], d['roofline']['achieved']); print(d['esia_k1000']); print(d['cpu_baseline']['value'], d.get('philox_mode'))"
(time python bench.py --impl reference) > gpurun_out/s3r17_bench_ref.json 2> gpurun_out/s3r17_bench_ref.err; tail -4 gpurun_out/s3r17_bench_ref.err; cut -c1-300 gpurun_out/s3r17_bench_ref.json

#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_greedy.py tests/test_gpu_fullsize.py tests/test_gpu_interdiction.py tests/test_gpu_sharded.py tests/test_gpu_baseline.py tests/test_gpu_sampler.py -x -q -m gpu > gpurun_out/s3r5_tests.log 2>&1; tail -4 gpurun_out/s3r5_tests.log
echo "== esia stages c4"; REPS=3 NO_TOUCH=1 python tools/esia_stages.py c4 2>&1 | tail -2
REPS=1 NO_TOUCH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s3r5_c4_esia_launches.csv python tools/esia_stages.py c4 > gpurun_out/s3r5_ncu_stdout.txt 2>&1
python tools/launch_summary.py gpurun_out/s3r5_c4_esia_launches.csv 24
echo "== bench"; python bench.py --no-cpu-baseline --no-philox --no-suspension --steps 5 2>/dev/null > gpurun_out/s3r5_bench.json; python -c "
import json; d=json.loads(open('gpurun_out/s3r5_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['stage_ms'], d['e2e']); print(d['esia_k1000'])"
echo "== esia stages c2 k1000"; REPS=3 NO_TOUCH=1 python tools/esia_stages.py c2 1000 2>&1 | tail -1

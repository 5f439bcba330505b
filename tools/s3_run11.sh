#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_greedy.py tests/test_gpu_fullsize.py tests/test_gpu_interdiction.py tests/test_gpu_sharded.py tests/test_gpu_baseline.py -x -q -m gpu > gpurun_out/s3r11_tests.log 2>&1; tail -4 gpurun_out/s3r11_tests.log
REPS=3 NO_TOUCH=1 python tools/esia_stages.py c4 2>&1 | tail -1
REPS=1 NO_TOUCH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s3r11_c4_esia_launches.csv python tools/esia_stages.py c4 > gpurun_out/s3r11_ncu_stdout.txt 2>&1
python tools/launch_summary.py gpurun_out/s3r11_c4_esia_launches.csv 22
REPS=3 NO_TOUCH=1 python tools/esia_stages.py c2 1000 2>&1 | tail -1
REPS=3 NO_TOUCH=1 python tools/esia_stages.py c3 2>&1 | tail -1

#!/bin/bash
mkdir -p gpurun_out
REPS=1 NO_TOUCH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s3r10_c4_esia_launches.csv python tools/esia_stages.py c4 > gpurun_out/s3r10_ncu_stdout.txt 2>&1
python tools/launch_summary.py gpurun_out/s3r10_c4_esia_launches.csv 32

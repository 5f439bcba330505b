#!/bin/bash
mkdir -p gpurun_out
echo "== dense, hist 8"; REPS=2 NO_TOUCH=1 python tools/esia_stages.py c4 2>&1 | tail -1
echo "== legacy, hist 8"; HSAW_DENSE_MIN_BYTES=1152921504606846976 REPS=2 NO_TOUCH=1 python tools/esia_stages.py c4 2>&1 | tail -1
echo "== dense, hist 16"; HSAW_HIST_BITS=16 REPS=2 NO_TOUCH=1 python tools/esia_stages.py c4 2>&1 | tail -1
echo "== dense, hist 12"; HSAW_HIST_BITS=12 REPS=2 NO_TOUCH=1 python tools/esia_stages.py c4 2>&1 | tail -1
REPS=1 NO_TOUCH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s3r3_c4_esia_dense_launches.csv python tools/esia_stages.py c4 > gpurun_out/s3r3_ncu_stdout.txt 2>&1
python tools/launch_summary.py gpurun_out/s3r3_c4_esia_dense_launches.csv 30
HSAW_UPLOAD_THREADS=8 python bench.py --no-esia --no-cpu-baseline --no-philox --no-suspension --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['e2e'])"

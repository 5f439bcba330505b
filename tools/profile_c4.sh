#!/bin/bash
# ncu evidence for the HBM-bound regime (C4, fat layout): launch list of a short bench run and one
# `--set full` capture each of K1 (fat encode kernel), K2b and the compaction kernel.
# Run under gpurun from the repo root; outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
WL=${1:-c4}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/r02_${WL}_launches.csv \
  python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-suspension --no-philox > gpurun_out/r02_${WL}_launches_bench.json 2> gpurun_out/r02_${WL}_launches.err
echo "launch list rc=$?"
for K in encode distinct_kernel compact_pairs; do
  # launches 0..2 of each kernel are the warm-up steps, launch 3 is the timed step (K1: the
  # recording kernel; the instrumented stats pass and the Philox leg come later)
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -s 3 -c 1 -f -o gpurun_out/r02_${WL}_$K \
    python bench.py --workload $WL --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-esia --no-philox > /dev/null 2> gpurun_out/r02_${WL}_$K.err
  echo "$K rc=$?"
  ncu -i gpurun_out/r02_${WL}_$K.ncu-rep --page details --csv > gpurun_out/r02_${WL}_${K}_details.csv 2>/dev/null
  python tools/ncu_key.py gpurun_out/r02_${WL}_$K.ncu-rep > gpurun_out/r02_${WL}_${K}_key.txt 2>&1
done
ls -la gpurun_out | tail -20

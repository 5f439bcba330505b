#!/bin/bash
# ncu evidence for one bench workload: launch list of a short bench run and one `--set full`
# capture each of K1 (encode kernel), K2b (main pass) and the compaction kernel, all of the TIMED
# step (launch index 3 after three warm-up steps; K2b launches twice per step: main, mid).
# Run under gpurun from the repo root; outputs land in gpurun_out/.
#   tools/profile_c4.sh [c4|c2|c3] [prefix]
set -u
mkdir -p gpurun_out
WL=${1:-c4}
PFX=${2:-r02d}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/${PFX}_${WL}_launches.csv \
  python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-suspension --no-philox > gpurun_out/${PFX}_${WL}_launches_bench.json 2> gpurun_out/${PFX}_${WL}_launches.err
echo "launch list rc=$?"
for K in encode:3 distinct_kernel:6 compact_pairs:3; do
  NAME=${K%%:*}; SKIP=${K##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$NAME -s $SKIP -c 1 -f -o gpurun_out/${PFX}_${WL}_$NAME \
    python bench.py --workload $WL --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-esia --no-philox > /dev/null 2> gpurun_out/${PFX}_${WL}_$NAME.err
  echo "$NAME rc=$?"
  ncu -i gpurun_out/${PFX}_${WL}_$NAME.ncu-rep --page details --csv > gpurun_out/${PFX}_${WL}_${NAME}_details.csv 2>/dev/null
  python tools/ncu_key.py gpurun_out/${PFX}_${WL}_$NAME.ncu-rep > gpurun_out/${PFX}_${WL}_${NAME}_key.txt 2>&1
  echo "== ${WL}_$NAME"; head -12 gpurun_out/${PFX}_${WL}_${NAME}_key.txt
done
python tools/launch_summary.py gpurun_out/${PFX}_${WL}_launches.csv 24 > gpurun_out/${PFX}_${WL}_launches_summary.txt; head -16 gpurun_out/${PFX}_${WL}_launches_summary.txt

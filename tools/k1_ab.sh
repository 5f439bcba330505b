#!/bin/bash
# A/B of K1 variants on the bench workload: prints "<label> <HSAW/s> <ms/step> <K1 ms>" per run.
# usage: tools/k1_ab.sh "LABEL ENV=1 ENV2=x" ...   (run on the GPU box)
for spec in "$@"; do
  label=${spec%% *}; envs=${spec#* }; [ "$envs" = "$spec" ] && envs=""
  env $envs python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-esia 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$label', round(d['value']/1e6,1), round(d['ms_per_step'],3), round(r['kernel_avg_ms'],3), {k:round(v/5,2) for k,v in r['stage_ms'].items()})"
done

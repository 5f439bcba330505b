#!/bin/bash
# A/B of the pipelined chunks (stream.cu sample_range) on the bench workload (run on the GPU box):
#   tools/pipe_ab.sh [workload] "LABEL ENV=1 ENV2=x" ...
WL=${1:-c4}; shift
for spec in "$@"; do
  label=${spec%% *}; envs=${spec#* }; [ "$envs" = "$spec" ] && envs=""
  env $envs python bench.py --workload $WL --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-suspension --no-philox 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; e=d.get('esia') or {}
print('$label', round(d['value']/1e6,1), 'M/s step', round(d['ms_per_step'],3), 'K1', round(r['kernel_avg_ms'],3), 'x', r['launches_timed'], {k:round(v/5,2) for k,v in r['stage_ms'].items()}, 'esia', e.get('seconds_to_solution'), e.get('breakdown_s'), 'cov', e.get('coverage'), e.get('samples_used'))"
done

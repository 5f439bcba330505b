#!/bin/bash
mkdir -p gpurun_out
echo "== dense, L2_PERSIST=0"; HSAW_L2_PERSIST=0 REPS=2 NO_TOUCH=1 python tools/esia_stages.py c4 2>&1 | tail -1
echo "== dense, default"; REPS=2 NO_TOUCH=1 python tools/esia_stages.py c4 2>&1 | tail -1
echo "== bench L2_PERSIST=0"; HSAW_L2_PERSIST=0 python bench.py --no-esia --no-cpu-baseline --no-philox --no-suspension --no-e2e --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['stage_ms'])"
echo "== bench default"; python bench.py --no-esia --no-cpu-baseline --no-philox --no-suspension --no-e2e --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['stage_ms'])"

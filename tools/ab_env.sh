#!/bin/bash
# A/B of environment settings on the bench workload (device-timed ms/step), round-robin,
# 3 rounds.  Usage: bash tools/ab_env.sh "TQ_GROUPS=1" "TQ_GROUPS=2"
for round in 1 2 3; do
  for v in "$@"; do
    env $v python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-c5-geometry 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4))"
  done
done

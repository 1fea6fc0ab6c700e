#!/bin/bash
# A/B of env-selected variants on the bench workload: bash scripts/ab_env.sh "NAME:ENV=.. ENV=.." ...
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
for cfg in "$@"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 300 $B > gpurun_out/ab_$name.log 2>&1
  echo "$name rc=$? $(head -c 200 gpurun_out/ab_$name.log | grep -o '"value": [0-9.]*') project_ms=$(python -c "import json; d=json.loads(open('gpurun_out/ab_$name.log').readline()); print(round(d['stages']['project']['ms_per_step'],1))" 2>/dev/null)"
done

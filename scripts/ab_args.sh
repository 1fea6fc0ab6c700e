#!/bin/bash
# A/B of bench arguments: bash scripts/ab_args.sh "NAME:--arg v ..." ...
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
for cfg in "$@"; do
  name=${cfg%%:*}; args=${cfg#*:}
  timeout 300 $B $args > gpurun_out/ab_$name.log 2>&1
  echo "$name rc=$? $(head -c 200 gpurun_out/ab_$name.log | grep -o '"value": [0-9.]*')"
done

#!/bin/bash
# A/B of K6 / pipeline variants on the bench workload (GPU box), then one
# ncu --set full capture of K6 with source.  Outputs under gpurun_out/.
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
for cfg in "base:" "slots1:--slots 1" "pix2:GSR_PIX=2" "stages8:GSR_STAGES=8" "pix2s8:GSR_PIX=2 GSR_STAGES=8"; do
  name=${cfg%%:*}; rest=${cfg#*:}
  envs=""; args=""
  for t in $rest; do case $t in GSR_*) envs="$envs $t";; *) args="$args $t";; esac; done
  env $envs timeout 300 $B $args > gpurun_out/ab_$name.log 2>&1
  echo "$name rc=$? $(head -c 200 gpurun_out/ab_$name.log | grep -o '"value": [0-9.]*')"
done
ncu --set full --clock-control none --import-source on -k regex:k6_composite -s 20 -c 1 \
    -o gpurun_out/prof_k6 $B --slots 1 > gpurun_out/ncu_k6.log 2>&1
echo "ncu rc=$?"

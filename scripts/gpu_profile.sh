#!/bin/bash
# Usage (on the GPU box, via gpurun): bash scripts/gpu_profile.sh TAG [KERNEL_REGEX]
# 1) plain short bench run (must exit 0), 2) ncu launch list, 3) ncu --set full
#    on the top kernels.  Outputs under gpurun_out/.
TAG=${1:-r1}
KRE=${2:-"k6_composite|onesweep|k3_emit"}
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --slots ${SLOTS:-1}"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain_$TAG.log; exit 1; }
# skip bench.py's untimed counting step and the warm-up step (~513 launches
# each at c3): the listed window is the timed step
ncu --metrics gpu__time_duration.sum --clock-control none -s ${LSKIP:-1030} -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s ${FSKIP:-400} -c ${NCOUNT:-8} \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full capture rc=$?"
ls -la gpurun_out/

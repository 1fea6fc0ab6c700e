#!/bin/bash
# bash scripts/gpu_ncu_kernel.sh TAG REGEX [SKIP] [COUNT] : plain run, then ncu --set full on matching kernels
TAG=$1; KRE=$2; SKIP=${3:-10}; CNT=${4:-2}
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --slots ${SLOTS:-1}"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain_$TAG.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c $CNT -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"

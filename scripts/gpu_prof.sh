#!/bin/bash
# ncu --set full capture of one launch of kernel regex $KRE (after the same command exits 0 without ncu).
# Outputs: gpurun_out/prof_$TAG.ncu-rep
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS}"
$CMD > gpurun_out/plain_$TAG.log 2>&1; echo PLAIN $?
ncu --set full --clock-control none --import-source on -k regex:"${KRE}" -s ${SKIP:-10} -c ${COUNT:-1} -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo NCU_RC $?
tail -3 gpurun_out/ncu_$TAG.log

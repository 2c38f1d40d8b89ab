#!/bin/bash
# ncu evidence for one bench step (run under gpurun): a --set full capture of one HVP launch (source
# counters) and the launch list of one step.  Each ncu command follows the same plain command exiting 0.
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-variants"
TAG=${1:-r2}
KRE=${2:-k_hvp_sw}
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 10 -c 1 -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo NCU1 $?
$CMD > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo NCU2 $?

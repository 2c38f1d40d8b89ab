#!/bin/bash
# full ncu capture of one launch of $KRE + the launch list of one bench step (1 warmup), after the
# command exits 0 without ncu
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-variants ${BENCH_ARGS}"
$CMD > gpurun_out/plain_$TAG.log 2>&1; echo PLAIN $?
ncu --set full --clock-control none --import-source on -k regex:"${KRE}" -s ${SKIP:-10} -c 1 -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo NCU_RC $?
ncu --metrics gpu__time_duration.sum --clock-control none -s 3200 -c 3200 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncul_$TAG.log 2>&1; echo NCUL_RC $?

#!/bin/bash
# One GPU session: full bench, then (after the same short command exits 0 without ncu) an ncu
# --set full capture of one HVP launch and the launch list of one step.  Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
free -g | head -2; nproc; lscpu | grep -E "Model name|MHz" | head -3
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo BENCH_RC $?
tail -3 gpurun_out/bench_full.err
cat gpurun_out/bench_full.json
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_hvp -s 10 -c 1 -o gpurun_out/prof_hvp -f $CMD > gpurun_out/ncu_hvp.log 2>&1; echo NCU1 $?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 3300 -c 3300 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo NCU2 $?

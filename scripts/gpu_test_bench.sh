#!/bin/bash
# GPU parity tests, smoke, a short bench, then an ncu --set full capture of one HVP and one
# gradient launch (after the same command exits 0 without ncu).  Outputs in gpurun_out/.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST_RC $?
tail -5 gpurun_out/pytest_gpu.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo SMOKE_RC $?; tail -2 gpurun_out/smoke.log
python bench.py --no-e2e ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH_RC $?
tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
if [ "${PROFILE:-1}" = "1" ]; then
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_hvp|k_grad" -s 12 -c 2 -o gpurun_out/prof -f $CMD > gpurun_out/ncu.log 2>&1; echo NCU_RC $?
fi

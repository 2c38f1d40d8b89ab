#!/bin/bash
# Round-end style session: GPU tests, smoke, the default bench line, then (after the same command
# exits 0 without ncu) one ncu --set full capture of the HVP and the launch list of one step.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST_RC $?; tail -2 gpurun_out/pytest_gpu.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo SMOKE_RC $?; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_round.json 2> gpurun_out/bench_round.err; echo BENCH_RC $?; cat gpurun_out/bench_round.json
if [ "${PROFILE:-1}" = "1" ]; then
TAG=${TAG:-round} KRE=k_hvp_sw bash scripts/gpu_prof2.sh
fi

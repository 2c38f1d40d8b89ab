#!/bin/bash
# Round-2 closing evidence on one B200 (run under gpurun): GPU tests, smoke, the driver-protocol bench,
# then the ncu captures (each after the same plain command exited 0): the fp64 HVP (--set full), the
# launch list of one step, and the fp32 HVP (--set full).  Outputs in gpurun_out/.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo PYTEST_RC $? >> gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo SMOKE_RC $? >> gpurun_out/final_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo BENCH_RC $? >> gpurun_out/final_bench.err
bash scripts/gpu_prof_r2.sh final k_hvp_sw > gpurun_out/final_prof.log 2>&1
C32="python bench.py --precision f32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-variants"
$C32 > gpurun_out/plain_f32.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_hvp_sw -s 10 -c 1 -o gpurun_out/prof_final_f32 -f $C32 > gpurun_out/ncu_final_f32.log 2>&1; echo NCU3 $? >> gpurun_out/final_prof.log
tail -2 gpurun_out/final_pytest.log; tail -1 gpurun_out/final_smoke.log; tail -1 gpurun_out/final_bench.err; cat gpurun_out/final_prof.log

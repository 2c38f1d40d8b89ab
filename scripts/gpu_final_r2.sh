#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): GPU tests, smoke, the driver-protocol bench, and the
# ncu captures (each after the same plain command exited 0).  Outputs in gpurun_out/.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo PYTEST_RC $? >> gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo SMOKE_RC $? >> gpurun_out/final_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo BENCH_RC $? >> gpurun_out/final_bench.err
bash scripts/gpu_prof_r2.sh final k_hvp_sw > gpurun_out/final_prof.log 2>&1

#!/bin/bash
# Round-2 physics / decomposition runs on one B200 (run under gpurun); outputs in gpurun_out/.
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-variants"
for v in 0 1; do
  timeout 300 $B --slabs 8 --cg-variant $v > gpurun_out/slab8_v$v.json 2> gpurun_out/slab8_v$v.err
done
timeout 300 $B --slabs 1 --cg-variant 1 > gpurun_out/slab1_v1.json 2> gpurun_out/slab1_v1.err
INCL_VERBOSE=1 timeout 1200 python scripts/inclusion_dual.py --protocol dynamic --ratio 2 --inv-h 64 --solver tol \
  --k-max 200 > gpurun_out/incl_dyn_tol.log 2>&1; echo rc=$? >> gpurun_out/incl_dyn_tol.log
timeout 1500 python scripts/cantilever_master.py --mode curve --dxb 0.0125 --psd 1 --guess 0 --rtol 1e-6 \
  --gammas 0.03 0.0675 0.152 0.342 0.769 1.15 1.73 2.6 3.0 4.0 6.0 9.0 13.5 20.0 26.8 \
  > gpurun_out/cant_psd.log 2>&1; echo rc=$? >> gpurun_out/cant_psd.log

#!/bin/bash
# Round-2 physics runs on one B200 (run under gpurun); outputs in gpurun_out/.
mkdir -p gpurun_out
INCL_VERBOSE=1 timeout 2400 python scripts/inclusion_dual.py --protocol dynamic --ratio 2 --inv-h 64 --solver tol \
  --k-max 200 > gpurun_out/incl_dyn_tol3.log 2>&1; echo rc=$? >> gpurun_out/incl_dyn_tol3.log
timeout 2400 python scripts/cantilever_master.py --mode curve --dxb 0.0125 --psd 1 --guess 0 --rtol 1e-6 --max-newton 300 \
  --gammas 0.03 0.0675 0.152 0.342 0.769 1.15 1.73 2.2 2.6 2.8 3.0 3.25 3.5 3.8 4.1 4.4 4.75 5.1 5.5 6.0 6.5 7.0 7.5 \
  8.1 8.8 9.5 10.3 11.1 12.0 13.0 14.0 15.2 16.4 17.7 19.2 20.7 22.4 24.5 26.8 \
  > gpurun_out/cant_psd3.log 2>&1; echo rc=$? >> gpurun_out/cant_psd3.log

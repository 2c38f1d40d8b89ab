#!/bin/bash
# Round-2 physics runs on one B200 (run under gpurun); outputs in gpurun_out/.
mkdir -p gpurun_out
OSMPM_DEBUG_LS=1 timeout 900 python scripts/cantilever_master.py --mode curve --dxb 0.0125 --psd 1 --guess 0 --rtol 1e-6 \
  --max-newton 300 --gammas 1.15 1.73 2.2 2.6 2.8 > gpurun_out/cant_dbg.log 2>&1; echo rc=$? >> gpurun_out/cant_dbg.log
INCL_VERBOSE=1 timeout 2400 python scripts/inclusion_dual.py --protocol dynamic --ratio 2 --inv-h 64 --solver tol \
  --k-max 200 > gpurun_out/incl_dyn_tol4.log 2>&1; echo rc=$? >> gpurun_out/incl_dyn_tol4.log

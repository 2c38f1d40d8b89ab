#!/bin/bash
# A/B of two builds on one box: OSMPM_LIB=ab/libosmpm_prev.so against the in-tree library, interleaved.
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-variants $*"
for r in 1 2; do
  OSMPM_LIB=ab/libosmpm_prev.so timeout 300 $B > gpurun_out/ab_prev_$r.json 2>/dev/null
  timeout 300 $B > gpurun_out/ab_new_$r.json 2>/dev/null
done
for f in gpurun_out/ab_prev_*.json gpurun_out/ab_new_*.json; do
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],2), round(d['roofline']['avg_launch_ms'],4))"
done

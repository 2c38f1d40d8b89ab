#!/bin/bash
# A/B of library builds on one box (run under gpurun): the in-tree library against ab/libosmpm_<tag>.so
# for each tag in $TAGS, interleaved over two rounds; prints ms/step and the HVP launch average.
mkdir -p gpurun_out
B="python bench.py --steps ${STEPS:-3} --warmup 3 --no-e2e --no-cpu-baseline --no-variants ${BENCH_ARGS}"
for r in 1 2; do
  timeout 300 $B > gpurun_out/ab_base_$r.json 2>/dev/null
  for t in $TAGS; do OSMPM_LIB=ab/libosmpm_$t.so timeout 300 $B > gpurun_out/ab_${t}_$r.json 2>/dev/null; done
done
for f in gpurun_out/ab_base_*.json $(for t in $TAGS; do echo gpurun_out/ab_${t}_*.json; done); do
  python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],2), round(d['roofline']['avg_launch_ms'],4))" 2>/dev/null || echo "$f failed"
done

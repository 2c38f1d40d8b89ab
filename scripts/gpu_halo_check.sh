#!/bin/bash
# fused-halo checks on one B200: dist/parity tests, then 8-slab benches (fused, both variants; halo pass).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_halo.log 2>&1; echo RC $? >> gpurun_out/pytest_halo.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-variants"
for v in 0 1; do timeout 300 $B --slabs 8 --cg-variant $v > gpurun_out/slab8f_v$v.json 2> gpurun_out/slab8f_v$v.err; done
OSMPM_FUSED_HALO=0 timeout 300 $B --slabs 8 > gpurun_out/slab8p_v0.json 2> gpurun_out/slab8p_v0.err
for f in slab8f_v0 slab8f_v1 slab8p_v0; do
  python -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],1), {k: round(v,1) for k, v in d['kernel_ms_per_step'].items()})"
done

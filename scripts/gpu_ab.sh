#!/bin/bash
# A/B of the HVP variants: GPU parity tests (default variant), then the short bench with each variant.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST_RC $?
tail -4 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-sw tiled}; do
  OSMPM_HVP=$v timeout 900 python bench.py --no-e2e --no-cpu-baseline --steps 2 ${BENCH_ARGS} > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
  echo BENCH_$v $?; tail -2 gpurun_out/bench_$v.err
  python -c "import json; d=json.load(open('gpurun_out/bench_$v.json')); print('$v', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['kernel_ms_per_step'])"
done

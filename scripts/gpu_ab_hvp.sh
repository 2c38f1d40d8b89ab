#!/bin/bash
# HVP A/B on C5 (run under gpurun): GPU parity tests, then the bench with the fp32 variant
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_hvp.log 2>&1; echo PYTEST_RC $?
tail -3 gpurun_out/pytest_hvp.log
fi
python bench.py --steps ${STEPS:-3} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_hvp.json 2> gpurun_out/ab_hvp.err; echo "BENCH rc=$?"
python - <<'PY'
import json
try:
    d=json.load(open("gpurun_out/ab_hvp.json"))
    print("f64", round(d["ms_per_step"],2), "hvp", round(d["roofline"]["avg_launch_ms"],4), "frac", round(d["roofline"]["frac"],4), {k: round(v,2) for k,v in d["kernel_ms_per_step"].items()})
    v=d["variants"]["f32"]; print("f32", round(v["ms_per_step"],2), "hvp", round(v["roofline"]["avg_launch_ms"],4), "frac", round(v["roofline"]["frac"],4))
except Exception as e:
    print("ERR", e); print(open("gpurun_out/ab_hvp.err").read()[-2000:])
PY

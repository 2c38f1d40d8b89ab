#!/bin/bash
# A/B of the PCG variants on C5 (run under gpurun): standard, single-reduction unfused, fused (R25)
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_cg.log 2>&1; echo PYTEST_RC $?
tail -3 gpurun_out/pytest_cg.log
fi
B="python bench.py --steps ${STEPS:-3} --warmup 3 --no-e2e --no-cpu-baseline --no-variants"
run() { tag=$1; shift; env "$@" $B > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; echo "$tag rc=$?"; }
for spec in ${RUNS:-"cg0:--cg-variant=0 cg1:--cg-variant=1"}; do
  tag=${spec%%:*}; args=${spec#*:}; envs=""
  IFS=',' read -ra parts <<< "$args"
  cmdargs=""; for p in "${parts[@]}"; do case $p in --*) cmdargs="$cmdargs ${p/=/ }";; *) envs="$envs $p";; esac; done
  env $envs $B $cmdargs > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; echo "$tag rc=$?"
  python - "$tag" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/ab_{f}.json"))
    print(f, round(d["ms_per_step"],2), "hvp", round(d["roofline"]["avg_launch_ms"],4), {k: round(v,2) for k,v in d["kernel_ms_per_step"].items()}, d["config"]["solve_stats_last_step"])
except Exception as e:
    print(f, "ERR", e); print(open(f"gpurun_out/ab_{f}.err").read()[-1500:])
PY
done

# A/B of HVP variants / launch modes: "name:ENV=VAL ..." pairs in $CASES
for c in ${CASES:-"sw:OSMPM_HVP=sw" "swfull:OSMPM_HVP=sw OSMPM_SW_FULLGRID=1"}; do
  name=${c%%:*}; envs=${c#*:}
  env $envs python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/ab_$name.json 2>gpurun_out/ab_$name.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$name.json')); print('$name', round(d['ms_per_step'],1), round(d['roofline']['avg_launch_ms'],4), round(sum(d['kernel_ms_per_step'].values()),1))"
done

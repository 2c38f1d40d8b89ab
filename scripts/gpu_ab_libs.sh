# A/B of library builds: "name:libpath" pairs in $LIBS; bench only
for c in $LIBS; do
  name=${c%%:*}; lib=${c#*:}
  OSMPM_LIB=$lib python bench.py --no-e2e --no-cpu-baseline --steps 2 ${BENCH_ARGS} > gpurun_out/ab_$name.json 2>gpurun_out/ab_$name.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$name.json')); print('$name', round(d['value']/1e6,3), round(d['ms_per_step'],1), round(d['roofline']['avg_launch_ms'],4), {k: round(v,1) for k,v in d['kernel_ms_per_step'].items()})"
done

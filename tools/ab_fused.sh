# A/B of fused-step variants: tests on the default build, then the bench per variant
timeout 600 python -m pytest tests -m gpu -x -q -k "bruss or nccl or multiinstance or ark or numerics" > gpurun_out/t_br.log 2>&1; tail -1 gpurun_out/t_br.log
for v in default ${VARIANTS}; do
  if [ $v = default ]; then unset SUNBW_LIB; else export SUNBW_LIB=$PWD/build/$v/libsunbw.so; fi
  timeout 300 python bench.py --no-ops --no-cpu --steps 200 > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', round(d['ms_per_step'],4), d['roofline']['achieved'], {k:v['us_avg'] for k,v in d['kernels'].items()})" 2>&1 | cut -c1-250
done

SUNBW_LIB=$PWD/build/var_m6g/libsunbw.so timeout 600 python -m pytest tests/test_gpu_bruss.py -x -q -p no:cacheprovider > gpurun_out/t_m6g.log 2>&1; tail -1 gpurun_out/t_m6g.log
SUNBW_LIB=$PWD/build/var_g5/libsunbw.so timeout 600 python -m pytest tests/test_gpu_bruss.py -x -q -p no:cacheprovider > gpurun_out/t_g5.log 2>&1; tail -1 gpurun_out/t_g5.log
for rep in 1 2; do
for v in default var_m6 var_g5 var_m6g; do
  if [ $v = default ]; then unset SUNBW_LIB; else export SUNBW_LIB=$PWD/build/$v/libsunbw.so; fi
  timeout 300 python bench.py --no-ops --no-cpu --steps 200 > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', round(d['ms_per_step'],4), d['roofline']['achieved'], {k:v['us_avg'] for k,v in d['kernels'].items()}, d['other_configs']['C1_64cells']['fused_steps_per_s'] if 'C1_64cells' in d['other_configs'] else '')" 2>&1 | cut -c1-250
done; done

# interleaved A/B of fused-step variants (VARIANTS), REPS rounds; fused kernel us per launch
SUNBW_LIB=$PWD/build/${TESTVAR}/libsunbw.so timeout 600 python -m pytest tests/test_gpu_bruss.py -x -q -p no:cacheprovider > gpurun_out/t_var.log 2>&1; echo "tests ${TESTVAR}: $(tail -1 gpurun_out/t_var.log)"
for rep in $(seq 1 ${REPS:-3}); do
for v in default ${VARIANTS}; do
  if [ $v = default ]; then unset SUNBW_LIB; else export SUNBW_LIB=$PWD/build/$v/libsunbw.so; fi
  timeout 300 python bench.py --no-ops --no-cpu --steps 200 > gpurun_out/ab_${v}_$rep.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$rep.json'));print('$rep $v', round(d['ms_per_step'],4), {k:v['us_avg'] for k,v in d['kernels'].items()})" 2>&1 | tail -1 | cut -c1-200
done; done

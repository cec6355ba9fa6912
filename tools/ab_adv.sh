# A/B of advection-stencil variants in the composed step (parity tests first)
python -m pytest tests/test_gpu_bruss.py -x -q -k "advection" > gpurun_out/t_adv.log 2>&1; tail -1 gpurun_out/t_adv.log
for v in default ${VARIANTS}; do
  if [ $v = default ]; then unset SUNBW_LIB; else export SUNBW_LIB=$PWD/build/$v/libsunbw.so; fi
  timeout 300 python bench.py --mode composed --no-ops --no-cpu --steps 30 > gpurun_out/abadv_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abadv_$v.json'));print('$v', round(d['ms_per_step'],4), d['kernels']['advection'])" 2>&1 | cut -c1-250
done

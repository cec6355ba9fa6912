SUNBW_LIB=$PWD/build/var_inv/libsunbw.so timeout 600 python -m pytest tests/test_gpu_contracted.py -q -p no:cacheprovider -x 2>&1 | tail -1
for i in 1 2; do
for v in default var_inv var_m6 var_inv_m6; do
  if [ $v = default ]; then L=""; else L=$PWD/build/$v/libsunbw.so; fi
  SUNBW_LIB=$L timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/ab_$v_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_$v_$i.json'));print('$v',d['kernels']['fused_newton']['us_avg'],round(d['value']/1e9,2))"
done; done

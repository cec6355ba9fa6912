timeout 900 python -m pytest tests/test_gpu_contracted.py tests/test_gpu_fused_tol.py -q -p no:cacheprovider -x 2>&1 | tail -1
for i in 1 2 3; do
  for v in new base; do
    if [ $v = new ]; then L=""; else L="SUNBW_LIB=$PWD/build/var_$v/libsunbw.so"; fi
    env $L timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/ab_${v}_${i}.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_${v}_${i}.json'));print('$v',d['kernels']['fused_newton']['us_avg'],round(d['value']/1e9,2))"
  done
done

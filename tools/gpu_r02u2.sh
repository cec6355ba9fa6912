SUNBW_LIB=$PWD/build/var_po/libsunbw.so timeout 900 python -m pytest tests/test_gpu_contracted.py tests/test_gpu_bruss.py -q -p no:cacheprovider -x 2>&1 | tail -1
for i in 1 2 3; do
  for v in def po; do
    if [ $v = def ]; then L=""; else L="SUNBW_LIB=$PWD/build/var_$v/libsunbw.so"; fi
    env $L timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/ab_${v}_${i}.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_${v}_${i}.json'));print('$v',d['kernels']['fused_newton']['us_avg'],round(d['value']/1e9,2))"
  done
done
for v in def po; do
  if [ $v = def ]; then L=""; else L="SUNBW_LIB=$PWD/build/var_$v/libsunbw.so"; fi
  env $L timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:fused_newton -s 3 -c 1 python bench.py --steps 5 --warmup 3 --no-ops --no-cpu 2>&1 | grep -E "dram__|gpu__time|lts__" | sed "s/^/$v /"
done

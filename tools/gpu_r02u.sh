SUNBW_LIB=$PWD/build/var_l2/libsunbw.so timeout 600 python -m pytest tests/test_gpu_contracted.py -q -p no:cacheprovider -x 2>&1 | tail -1
for i in 1 2 3; do
  timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/ab_def_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_def_$i.json'));print('default',d['kernels']['fused_newton']['us_avg'],round(d['value']/1e9,2))"
  SUNBW_LIB=$PWD/build/var_l2/libsunbw.so timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/ab_l2_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_l2_$i.json'));print('l2hint',d['kernels']['fused_newton']['us_avg'],round(d['value']/1e9,2))"
done
SUNBW_LIB=$PWD/build/var_l2/libsunbw.so timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fused_newton -s 3 -c 1 python bench.py --steps 5 --warmup 3 --no-ops --no-cpu 2>&1 | grep -E "dram__|gpu__time"
SUNBW_LIB=$PWD/build/var_l2/libsunbw.so timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fused_newton -s 3 -c 1 python bench.py --steps 5 --warmup 3 --no-ops --no-cpu --numerics exact 2>&1 | grep -E "dram__|gpu__time"

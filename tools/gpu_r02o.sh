timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_o.log 2>&1; tail -3 gpurun_out/pytest_gpu_o.log
for i in 1 2; do
  timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/o_$i.json 2>gpurun_out/o_$i.err
  python -c "import json;d=json.load(open('gpurun_out/o_$i.json'));print('HF',d['kernels']['fused_newton']['us_avg'],round(d['value']/1e9,2),d['roofline']['frac'])"
  timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu --numerics exact > gpurun_out/oe_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/oe_$i.json'));print('HF exact',d['kernels']['fused_newton']['us_avg'],round(d['value']/1e9,2))"
done
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fused_newton -s 3 -c 1 python bench.py --steps 5 --warmup 3 --no-ops --no-cpu 2>&1 | grep -E "dram__|gpu__time"

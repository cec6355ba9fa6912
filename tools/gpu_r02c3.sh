timeout 900 python -m pytest tests/test_gpu_bruss.py tests/test_gpu_contracted.py tests/test_gpu_multiinstance.py -q -p no:cacheprovider -x 2>&1 | tail -1
for i in 1 2 3; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-ops --no-cpu > gpurun_out/c3_$i.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/c3_$i.json').read().strip().splitlines()[-1]);k=d['kernels']['fused_newton'];print('steps20', k['us_avg'], k['share'], round(d['ms_per_step']*1e3,1), round(d['value']/1e9,2), d['gpu_launches'])"
done

set -x
timeout 900 python -m pytest tests/test_gpu_bruss.py tests/test_gpu_contracted.py tests/test_gpu_multirank_flags.py tests/test_gpu_ark.py -q -x -p no:cacheprovider 2>&1 | tail -5
for i in 1 2; do
SUNBW_KWALK=0 timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/b_lin$i.json 2>gpurun_out/b_lin$i.err
SUNBW_KWALK=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/b_walk$i.json 2>gpurun_out/b_walk$i.err
done
for f in gpurun_out/b_lin*.json gpurun_out/b_walk*.json; do python -c "import json,sys;d=json.load(open('$f'));print('$f',d['kernels']['fused_newton']['us_avg'],d['kernels']['fused_newton']['share'],round(d['value']/1e9,2))"; done
timeout 20 python bench.py --steps 20 --warmup 5 --no-ops --no-cpu > gpurun_out/b_20.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/b_20.json'));print('steps20',d['kernels'],d['value']/1e9,d['e2e']['value']/1e9)"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_newton -s 3 -c 1 -o gpurun_out/prof_walk python bench.py --steps 5 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
ls gpurun_out

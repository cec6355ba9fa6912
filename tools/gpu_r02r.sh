./build/tile_streams
timeout 900 python -m pytest tests/test_gpu_bruss.py -q -p no:cacheprovider -x -k "C1 or tol or graph" 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-ops --no-cpu > gpurun_out/b20_$i.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b20_$i.json'));print('steps20',d['kernels'],round(d['value']/1e9,2),d['gpu_launches'])"; done

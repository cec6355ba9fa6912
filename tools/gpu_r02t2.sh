timeout 600 python -m pytest tests/test_gpu_ark.py -q -p no:cacheprovider -x 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 --no-ops > gpurun_out/bench_t2.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/bench_t2.json').read().strip().splitlines()[-1]);c=d['cpu_baseline'];print('cpu_baseline',c['value'],c['sample'])"
for i in 1 2; do timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_t2_$i.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/ref_t2_$i.json').read().strip().splitlines()[-1]);print('ref',d['value'])"; done

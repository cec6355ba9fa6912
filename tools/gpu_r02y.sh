timeout 900 python -m pytest tests/test_gpu_two_step.py -q -p no:cacheprovider -x 2>&1 | tail -1
timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/two_1.json 2>gpurun_out/two_1.err
python -c "import json;d=json.load(open('gpurun_out/two_1.json'));print('two-step',d['kernels'],round(d['value']/1e9,2),d['ms_per_step'])"

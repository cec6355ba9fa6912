set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_contracted.py -q -x -p no:cacheprovider 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_bruss.py -q -x -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -5
timeout 300 python bench.py --steps 100 --warmup 5 --no-ops --no-cpu > gpurun_out/b_ct.json 2>gpurun_out/b_ct.err; python -c "import json;d=json.load(open('gpurun_out/b_ct.json'));print(d['kernels'],d['value'],d['roofline']['frac'])"
timeout 300 python bench.py --steps 100 --warmup 5 --no-ops --no-cpu --numerics exact > gpurun_out/b_ex.json 2>gpurun_out/b_ex.err; python -c "import json;d=json.load(open('gpurun_out/b_ex.json'));print(d['kernels'],d['value'],d['roofline']['frac'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_newton -s 3 -c 1 -o gpurun_out/prof_ct python bench.py --steps 5 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
ls gpurun_out

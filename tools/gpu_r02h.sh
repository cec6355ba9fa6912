set -x
timeout 900 python -m pytest tests/test_gpu_ark.py tests/test_gpu_fused_tol.py tests/test_gpu_bruss.py tests/test_gpu_contracted.py -q -p no:cacheprovider > gpurun_out/pytest_h.log 2>&1; tail -15 gpurun_out/pytest_h.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; python -c "import json;d=json.load(open('gpurun_out/bench_default.json'));o=d['other_configs'];print(json.dumps({k:o[k] for k in ('C3_adaptive_ARK','C3_adaptive_ARK_fused','C5_tolerance_mode')}));print(d['value'],d['kernels'])"
tail -3 gpurun_out/bench_default.err

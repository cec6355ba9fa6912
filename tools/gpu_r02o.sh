timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
grep -E "FAILED|Error" gpurun_out/pytest_gpu.log | head
timeout 300 python tools/ark_bench.py

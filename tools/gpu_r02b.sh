set -x
timeout 900 python -m pytest tests/test_gpu_contracted.py -q -p no:cacheprovider 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_bruss.py tests/test_gpu_numerics.py -q -x -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -3

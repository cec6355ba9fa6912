SUNBW_LIB=$PWD/build/var_cnt/libsunbw.so timeout 300 python tools/count_exact.py > gpurun_out/count_exact.log 2>&1; tail -5 gpurun_out/count_exact.log
timeout 600 python -m pytest tests/test_gpu_nvector.py -q -p no:cacheprovider -k beyond > gpurun_out/t_beyond.log 2>&1; tail -3 gpurun_out/t_beyond.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log

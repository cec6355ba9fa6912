SUNBW_LIB=$PWD/build/var_minb6/libsunbw.so timeout 600 python -m pytest tests/test_gpu_bruss.py -x -q -p no:cacheprovider > gpurun_out/t_minb6.log 2>&1; tail -1 gpurun_out/t_minb6.log
VARIANTS="var_minb6 var_minb6h" bash tools/ab_l2.sh

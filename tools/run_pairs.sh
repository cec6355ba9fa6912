timeout 900 python -m pytest tests/test_gpu_bruss.py tests/test_gpu_nccl.py -x -q -p no:cacheprovider > gpurun_out/t_pairs.log 2>&1; tail -2 gpurun_out/t_pairs.log
TESTVAR=var_nopairs VARIANTS="var_nopairs" REPS=3 bash tools/ab_rep.sh
for v in default var_nopairs; do
  if [ $v = default ]; then unset SUNBW_LIB; else export SUNBW_LIB=$PWD/build/$v/libsunbw.so; fi
  echo "ncu $v"; timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:fused_newton -s 5 -c 2 --csv python bench.py --steps 3 --warmup 3 --no-ops --no-cpu 2>/dev/null | grep -v "^==" | awk -F'","' '{print $(NF-2), $NF}' | tail -8
done

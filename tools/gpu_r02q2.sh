SUNBW_ARK_L2=1 timeout 900 python -m pytest tests/test_gpu_ark.py -q -p no:cacheprovider -x 2>&1 | tail -1
for i in 1 2; do for m in 0 1 2; do
  echo -n "l2=$m "; SUNBW_ARK_L2=$m timeout 300 python tools/ark_bench.py
done; done
for m in 0 1 2; do
SUNBW_ARK_L2=$m timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_ark_tile -s 8 -c 4 python tools/ark_profile.py 128 0.002 2>&1 | grep -E "dram__|gpu__time" | awk -v m=$m '{printf "l2=%s %s %s %s\n", m, $1, $2, $3}'
done

# ncu DRAM bytes + time of the fused step for the default build and VARIANTS (2 launches each)
for v in default ${VARIANTS}; do
  if [ $v = default ]; then unset SUNBW_LIB; else export SUNBW_LIB=$PWD/build/$v/libsunbw.so; fi
  echo "== $v"
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:fused_newton -s 5 -c 2 --csv python bench.py --steps 3 --warmup 3 --no-ops --no-cpu 2>/dev/null | grep -v "^==" | python -c "import csv,sys; [print(r[-3], r[-2], r[-1]) for r in csv.reader(sys.stdin) if len(r) > 3][1:]"
done

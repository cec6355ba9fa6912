# A/B of fused-step L2 variants: bench + ncu DRAM bytes of one fused launch per variant
for v in default ${VARIANTS}; do
  if [ $v = default ]; then unset SUNBW_LIB; else export SUNBW_LIB=$PWD/build/$v/libsunbw.so; fi
  timeout 300 python bench.py --no-ops --no-cpu --steps 200 > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', round(d['ms_per_step'],4), d['roofline']['achieved'], {k:v['us_avg'] for k,v in d['kernels'].items()})" 2>&1 | cut -c1-250
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:fused_newton -s 5 -c 2 --csv python bench.py --steps 3 --warmup 3 --no-ops --no-cpu 2>/dev/null | grep -v "^==" | cut -d, -f12- | tail -8
done

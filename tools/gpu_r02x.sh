for i in 1 2; do
  SUNBW_TWO_STEP=0 timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/one_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/one_$i.json'));print('one-step',d['kernels'],round(d['value']/1e9,2),d['ms_per_step'])"
  timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/two_$i.json 2>gpurun_out/two_$i.err
  python -c "import json;d=json.load(open('gpurun_out/two_$i.json'));print('two-step',d['kernels'],round(d['value']/1e9,2),d['ms_per_step'])"
done
tail -3 gpurun_out/two_1.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-ops --no-cpu > gpurun_out/two_20.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/two_20.json'));print('two-step@20',d['kernels'],round(d['value']/1e9,2),d['ms_per_step'])"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fused_newton2 -s 2 -c 1 -o /tmp/prof2 python bench.py --steps 6 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof2.ncu-rep > gpurun_out/ncu_summary_2step.txt; python tools/ncu_stalls.py /tmp/prof2.ncu-rep > gpurun_out/ncu_stalls_2step.txt 2>&1; cat gpurun_out/ncu_summary_2step.txt; head -16 gpurun_out/ncu_stalls_2step.txt

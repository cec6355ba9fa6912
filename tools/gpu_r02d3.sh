timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "timing or kernel_times or bruss or contracted" -x 2>&1 | tail -1
for i in 1 2; do for st in 20 200; do
  timeout 600 python bench.py --steps $st --warmup 5 --no-ops --no-cpu > gpurun_out/d3_${st}_$i.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/d3_${st}_$i.json').read().strip().splitlines()[-1]);k=d['kernels']['fused_newton'];print('steps $st', k['us_avg'], k['launches'], k['share'], round(d['ms_per_step']*1e3,1), round(d['value']/1e9,2), d['roofline']['frac'])"
done; done
timeout 600 python tools/step_gaps_cupti.py 2>&1 | grep timing=

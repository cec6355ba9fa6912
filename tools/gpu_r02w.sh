timeout 900 python -m pytest tests/test_gpu_two_step.py -q -p no:cacheprovider -x 2>&1 | tail -5
for i in 1 2; do
  SUNBW_TWO_STEP=0 timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/one_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/one_$i.json'));print('one-step',d['kernels'],round(d['value']/1e9,2),d['ms_per_step'])"
  timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/two_$i.json 2>gpurun_out/two_$i.err
  python -c "import json;d=json.load(open('gpurun_out/two_$i.json'));print('two-step',d['kernels'],round(d['value']/1e9,2),d['ms_per_step'])"
done
tail -3 gpurun_out/two_1.err
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_ark.py -q -p no:cacheprovider -k "C3_shape and shape1" > gpurun_out/san_race_ark.log 2>&1; echo "racecheck ark rc=$?" >> gpurun_out/san_race_ark.log; tail -3 gpurun_out/san_race_ark.log

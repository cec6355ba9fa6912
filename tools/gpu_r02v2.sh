timeout 900 python -m pytest tests/test_gpu_fused_tol.py tests/test_gpu_multirank_flags.py tests/test_gpu_contracted.py -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_v2.json 2> gpurun_out/bench_v2.err; tail -2 gpurun_out/bench_v2.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_v2.json").read().strip().splitlines()[-1])
print(d["value"]/1e9, json.dumps(d["other_configs"].get("C5_tolerance_mode")))
PY

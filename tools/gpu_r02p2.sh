timeout 900 python -m pytest tests/test_gpu_fused_tol.py tests/test_gpu_multirank_flags.py -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_p2.json 2> gpurun_out/bench_p2.err; tail -2 gpurun_out/bench_p2.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_p2.json").read().strip().splitlines()[-1])
print(d["value"]/1e9, d["kernels"])
for k in ("C5_tolerance_mode","C3_adaptive_ARK_fused","C3_3D_128cubed"):
    print(k, json.dumps(d["other_configs"].get(k)))
print(json.dumps(d["e2e"])[:300])
PY

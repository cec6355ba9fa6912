timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err; tail -3 gpurun_out/bench_k.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_k.json").read().strip().splitlines()[-1])
print(d["value"]/1e9, d["ms_per_step"], json.dumps(d["e2e"]))
print(json.dumps(d["other_configs"].get("C3_adaptive_ARK_fused")), json.dumps(d["other_configs"].get("C3_adaptive_ARK")))
PY

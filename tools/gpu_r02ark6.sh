timeout 900 python -m pytest tests/test_gpu_ark.py tests/test_gpu_multirank_flags.py -q -p no:cacheprovider -x 2>&1 | tail -4
for i in 1 2; do for gr in 1 0; do for cfg in 3331 3333; do
  echo -n "graph=$gr cfg=$cfg "; SUNBW_ARK_GRAPH=$gr SUNBW_ARK_CFG=$cfg timeout 300 python tools/ark_bench.py
done; done; done
SUNBW_ARK_CFG=3333 timeout 300 python tools/ark_timeline.py > gpurun_out/ark_tl_g.json 2>&1
python - <<'PY'
import json
d=json.load(open("gpurun_out/ark_tl_g.json"))
print(d["span_us"], d["us_per_attempt"], {k:(v["count"],v["us_avg"]) for k,v in d["kernels"].items()})
print("  gaps", {k:(v["count"],v["us_avg"]) for k,v in list(d["gaps"].items())[:6]})
PY

timeout 900 python -m pytest tests/test_gpu_ark.py -q -p no:cacheprovider -x 2>&1 | tail -2
for cfg in 1111 3331 3333 2221 4441 2222; do
  SUNBW_ARK_CFG=$cfg timeout 300 python tools/ark_timeline.py > gpurun_out/ark_tl_$cfg.json 2>/dev/null
  python - $cfg <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/ark_tl_{sys.argv[1]}.json"))
print(sys.argv[1], d["span_us"], d["us_per_attempt"], {k:v["us_avg"] for k,v in d["kernels"].items()})
PY
done

timeout 900 python -m pytest tests/test_gpu_ark.py tests/test_gpu_multirank_flags.py -q -p no:cacheprovider -x 2>&1 | tail -4
for i in 1 2; do for cfg in 3333 3334 3331; do
  echo -n "cfg=$cfg "; SUNBW_ARK_CFG=$cfg timeout 300 python tools/ark_bench.py
done; done
SUNBW_ARK_CFG=3333 timeout 300 python tools/ark_timeline.py > gpurun_out/ark_tl_c.json 2>/dev/null
python - <<'PY'
import json
d=json.load(open("gpurun_out/ark_tl_c.json"))
print(d["span_us"], d["us_per_attempt"], {k:(v["count"],v["us_avg"]) for k,v in d["kernels"].items()})
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ark_tile -s 8 -c 4 -o gpurun_out/prof_ark3 python tools/ark_profile.py 128 0.002 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_ark3.ncu-rep > gpurun_out/ncu_summary_ark3.txt 2>&1; grep -E "kernel|time_dur|dram__bytes|issue_active|warps_active" gpurun_out/ncu_summary_ark3.txt

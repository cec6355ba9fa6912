timeout 900 python -m pytest tests/test_gpu_ark.py tests/test_gpu_multirank_flags.py -q -p no:cacheprovider -x 2>&1 | tail -4
for cfg in 3331 3333; do
  SUNBW_ARK_CFG=$cfg timeout 300 python tools/ark_timeline.py > gpurun_out/ark_tl_$cfg.json 2>gpurun_out/ark_tl_$cfg.err
  python - $cfg <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/ark_tl_{sys.argv[1]}.json"))
print(sys.argv[1], d["span_us"], d["us_per_attempt"], d["stats"]["newton_iters"], {k:(v["count"],v["us_avg"]) for k,v in d["kernels"].items()})
print("  gaps", {k:(v["count"],v["us_avg"]) for k,v in list(d["gaps"].items())[:6]})
PY
done
timeout 300 python tools/ark_bench.py
timeout 300 python tools/ark_bench.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ark_tile -s 8 -c 4 -o gpurun_out/prof_ark2 python tools/ark_profile.py 128 0.002 > gpurun_out/prof_ark2.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_ark2.ncu-rep > gpurun_out/ncu_summary_ark2.txt 2>&1; grep -E "kernel|time_dur|dram__bytes|issue_active|warps_active|fp64.avg" gpurun_out/ncu_summary_ark2.txt

timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_final2.log 2>&1; tail -1 gpurun_out/pytest_gpu_final2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1; tail -1 gpurun_out/smoke_final2.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; tail -2 gpurun_out/bench_final2.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_final2.json 2>&1
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_final2.json").read().strip().splitlines()[-1])
print(d["value"]/1e9, d["kernels"], d["roofline"]["frac"], d["roofline"]["traffic"], d["e2e"]["value"]/d["value"], d["cpu_baseline"]["value"])
r=json.loads(open("gpurun_out/bench_ref_final2.json").read().strip().splitlines()[-1]); print("ref", r["value"])
PY

timeout 1200 python -m pytest tests/test_gpu_ark.py tests/test_gpu_bruss.py tests/test_gpu_fused_tol.py tests/test_gpu_multirank_flags.py -q -p no:cacheprovider -x > gpurun_out/pytest_m.log 2>&1; tail -15 gpurun_out/pytest_m.log
timeout 300 python tools/ark_bench.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ark_launches.csv python tools/ark_profile.py 128 0.002 > gpurun_out/ark_prof.log 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/ark_launches.csv')))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[hdr+1:]:
    if len(r)>iv: d[r[ik][:50]].append(float(r[iv].replace(',','')))
for k,v in d.items(): print(f"{k:50s} n={len(v):4d} avg={sum(v)/len(v)/1e3:8.1f} us")
PY

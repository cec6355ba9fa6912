timeout 900 python -m pytest tests/test_gpu_ark.py -q -p no:cacheprovider 2>&1 | tail -2
for ks in 1 2; do SUNBW_ARK_KS=$ks timeout 300 python tools/ark_bench.py; done
timeout 300 python tools/ark_bench.py --composed
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

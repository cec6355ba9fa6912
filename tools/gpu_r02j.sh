timeout 900 python -m pytest tests/test_gpu_ark.py -q -p no:cacheprovider > gpurun_out/pytest_ark.log 2>&1; tail -5 gpurun_out/pytest_ark.log
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
timeout 300 ncu --set full --clock-control none -k regex:k_ark_tile -s 8 -c 4 -o /tmp/ark python tools/ark_profile.py 128 0.002 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ark.ncu-rep > gpurun_out/ark_ncu_summary.txt 2>&1; grep -E "kernel|duration|dram__bytes|throughput|warps_active|issue" gpurun_out/ark_ncu_summary.txt

timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ark_launches.csv python tools/ark_profile.py 128 0.002 > gpurun_out/ark_prof.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_ark_stage -s 8 -c 4 -o /tmp/ark python tools/ark_profile.py 128 0.002 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ark.ncu-rep > gpurun_out/ark_ncu_summary.txt 2>&1
python tools/ncu_stalls.py /tmp/ark.ncu-rep 2097152 > gpurun_out/ark_ncu_stalls.txt 2>&1
ncu -i /tmp/ark.ncu-rep --page details --csv > gpurun_out/ark_details.csv 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/ark_launches.csv')))
hdr=None
for i,r in enumerate(rows):
    if 'Kernel Name' in r: hdr=i;break
h=rows[hdr]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
import collections
d=collections.defaultdict(list)
for r in rows[hdr+1:]:
    if len(r)>iv: d[r[ik][:60]].append(float(r[iv].replace(',','')))
for k,v in d.items(): print(f"{k:60s} n={len(v):4d} avg={sum(v)/len(v)/1e3:8.1f} us")
PY

timeout 400 ncu --set full --clock-control none --import-source on -k regex:fused_newton -s 3 -c 1 -o gpurun_out/prof_ct python bench.py --steps 5 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fused_newton -s 3 -c 1 -o gpurun_out/prof_ex python bench.py --steps 5 --warmup 3 --no-ops --no-cpu --numerics exact > /dev/null 2>&1
python tools/traffic_json.py gpurun_out/prof_ct.ncu-rep gpurun_out/prof_ex.ncu-rep > gpurun_out/traffic.log 2>&1; cp profiles/ncu_traffic.json gpurun_out/
python tools/ncu_summary.py gpurun_out/prof_ct.ncu-rep > gpurun_out/ncu_summary_ct.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof_ex.ncu-rep > gpurun_out/ncu_summary_ex.txt 2>&1
python tools/ncu_stalls.py gpurun_out/prof_ct.ncu-rep > gpurun_out/ncu_stalls_ct.txt 2>&1
rm -f gpurun_out/prof_ex.ncu-rep
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_fused.csv python bench.py --steps 5 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 300 gpurun_out/bench_default.json

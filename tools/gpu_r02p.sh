set -x
timeout 300 python tools/halo_overlap.py 8 64 > gpurun_out/halo_overlap.json 2> gpurun_out/halo_overlap.err; cat gpurun_out/halo_overlap.json; tail -3 gpurun_out/halo_overlap.err
SUNBW_PEER_HALO=0 timeout 300 python tools/halo_overlap.py 8 64 > gpurun_out/halo_overlap_nccl_path.json 2>&1; cat gpurun_out/halo_overlap_nccl_path.json | tail -2
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fused_newton -s 3 -c 1 -o /tmp/prof_ct python bench.py --steps 5 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fused_newton -s 3 -c 1 -o /tmp/prof_ex python bench.py --steps 5 --warmup 3 --no-ops --no-cpu --numerics exact > /dev/null 2>&1
python tools/traffic_json.py /tmp/prof_ct.ncu-rep /tmp/prof_ex.ncu-rep > gpurun_out/traffic.log 2>&1; cp profiles/ncu_traffic.json gpurun_out/
python tools/ncu_summary.py /tmp/prof_ct.ncu-rep > gpurun_out/ncu_summary_ct.txt; python tools/ncu_summary.py /tmp/prof_ex.ncu-rep > gpurun_out/ncu_summary_ex.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 200 gpurun_out/bench_default.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_fused.csv python bench.py --steps 5 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
du -sh gpurun_out

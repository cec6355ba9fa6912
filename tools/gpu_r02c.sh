set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 400 gpurun_out/bench_default.json
timeout 300 python bench.py --steps 100 --warmup 5 --no-ops --no-cpu --numerics exact > gpurun_out/b_ex.json 2>gpurun_out/b_ex.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_fused.csv python bench.py --steps 5 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_newton -s 3 -c 1 -o gpurun_out/prof_ct python bench.py --steps 5 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
ls gpurun_out

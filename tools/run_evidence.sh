set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 300 gpurun_out/bench_default.json
timeout 300 python bench.py --mode composed --steps 100 --no-ops --no-cpu > gpurun_out/bench_composed.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_fused.csv python bench.py --steps 5 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_composed.csv python bench.py --mode composed --steps 2 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fused_newton -s 3 -c 1 -o gpurun_out/prof_fused python bench.py --steps 5 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_lu_solve|k_lu_factor|k_stream|k_reduce" -s 20 -c 6 -o gpurun_out/prof_composed python bench.py --mode composed --steps 2 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
[ -n "$SANITIZE" ] && timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_blockdiag.py -q -p no:cacheprovider -k "not 70001" > gpurun_out/sanitizer_memcheck.log 2>&1; echo memcheck rc=$? >> gpurun_out/sanitizer_memcheck.log; tail -3 gpurun_out/sanitizer_memcheck.log
[ -n "$SANITIZE" ] && timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_bruss.py -q -p no:cacheprovider -k "3D_fused_step_kernel or C1_fixed_K" > gpurun_out/sanitizer_racecheck.log 2>&1; echo racecheck rc=$? >> gpurun_out/sanitizer_racecheck.log; tail -3 gpurun_out/sanitizer_racecheck.log
ls -la gpurun_out

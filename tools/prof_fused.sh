timeout 400 ncu --set full --clock-control none --import-source on -k regex:fused_newton -s 3 -c 1 -o gpurun_out/prof_fused_cur python bench.py --steps 5 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1

timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_last.log 2>&1; tail -1 gpurun_out/pytest_gpu_last.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_last.log 2>&1; tail -1 gpurun_out/smoke_last.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ark_tile -s 8 -c 4 -o gpurun_out/prof_ark_last python tools/ark_profile.py 128 0.002 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_ark_last.ncu-rep > gpurun_out/ncu_summary_ark_last.txt 2>&1
timeout 300 python tools/ark_timeline.py > gpurun_out/ark_timeline_last.json 2>/dev/null
rm -f gpurun_out/prof_ark_last.ncu-rep.bak

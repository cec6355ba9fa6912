set -x
timeout 300 python tools/ark_timeline.py > gpurun_out/ark_timeline.json 2> gpurun_out/ark_timeline.err; head -c 3000 gpurun_out/ark_timeline.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/ark_launches.csv python tools/ark_profile.py 128 0.002 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ark_tile -s 8 -c 4 -o gpurun_out/prof_ark python tools/ark_profile.py 128 0.002 > gpurun_out/prof_ark.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_ark.ncu-rep > gpurun_out/ncu_summary_ark.txt 2>&1; cat gpurun_out/ncu_summary_ark.txt
python tools/ncu_stalls.py gpurun_out/prof_ark.ncu-rep > gpurun_out/ncu_stalls_ark.txt 2>&1; head -60 gpurun_out/ncu_stalls_ark.txt

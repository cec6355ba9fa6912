timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_ark_tile -s 8 -c 4 -o /tmp/ark python tools/ark_profile.py 128 0.002 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ark.ncu-rep > gpurun_out/ark_ncu_summary.txt 2>&1
python tools/ncu_stalls.py /tmp/ark.ncu-rep 2097152 > gpurun_out/ark_ncu_stalls.txt 2>&1
ncu -i /tmp/ark.ncu-rep --page details --csv > gpurun_out/ark_details.csv 2>&1
ncu -i /tmp/ark.ncu-rep --page source --csv --print-source sass -k regex:"k_ark_tile<1" > gpurun_out/ark_src1.csv 2>&1
ls -la gpurun_out

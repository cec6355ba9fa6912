for i in 1 2; do
for v in "0 0" "1 0" "1 1" "1 2" "1 26"; do set -- $v
SUNBW_KWALK=$1 SUNBW_KWALK_SEG=$2 timeout 300 python bench.py --steps 200 --warmup 5 --no-ops --no-cpu > gpurun_out/b_$1_$2_$i.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_$1_$2_$i.json'));print('walk=$1 seg=$2',d['kernels']['fused_newton']['us_avg'],round(d['value']/1e9,2))"
done; done
SUNBW_KWALK_SEG=1 timeout 600 ncu --set full --clock-control none -k regex:fused_newton -s 3 -c 1 -o gpurun_out/prof_walk1 python bench.py --steps 5 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1
SUNBW_KWALK=0 timeout 600 ncu --set full --clock-control none -k regex:fused_newton -s 3 -c 1 -o gpurun_out/prof_lin python bench.py --steps 5 --warmup 3 --no-ops --no-cpu > /dev/null 2>&1

SUNBW_ARK_PDL=1 timeout 600 python -m pytest tests/test_gpu_ark.py -q -p no:cacheprovider -x 2>&1 | tail -1
for i in 1 2 3; do for m in 0 1; do
  echo -n "pdl=$m "; SUNBW_ARK_PDL=$m timeout 300 python tools/ark_bench.py
done; done

for i in 1 2; do for sp in 1 2 4; do
  SUNBW_E2E_SPLIT=$sp timeout 600 python bench.py --steps 20 --warmup 5 --no-ops --no-cpu > gpurun_out/e2e_$sp.json 2>gpurun_out/e2e_$sp.err
  python -c "import json;d=json.loads(open('gpurun_out/e2e_$sp.json').read().strip().splitlines()[-1]);print('split $sp', round(d['e2e']['value']/1e9,2), round(d['e2e']['value']/d['value'],3), d['e2e']['ms'])"
done; done
tail -3 gpurun_out/e2e_4.err

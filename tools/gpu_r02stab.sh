for i in 1 2; do
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=300 > gpurun_out/pytest_stab_$i.log 2>&1; tail -1 gpurun_out/pytest_stab_$i.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_stab.log 2>&1; tail -1 gpurun_out/smoke_stab.log

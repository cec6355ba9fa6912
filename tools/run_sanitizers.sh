# compute-sanitizer on the GPU test subsets (small sizes), logs under gpurun_out/
set -x
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -p no:cacheprovider \
  tests/test_gpu_blockdiag.py tests/test_gpu_gmres.py tests/test_gpu_ark.py tests/test_gpu_numerics.py \
  -k "not 70001 and not 50_001 and not random" > gpurun_out/sanitizer_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/sanitizer_memcheck.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -p no:cacheprovider \
  tests/test_gpu_bruss.py -k "fused_step_kernel or multirank_driver or C1_fixed_K or linear_test" \
  > gpurun_out/sanitizer_memcheck_driver.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/sanitizer_memcheck_driver.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest -q -p no:cacheprovider \
  tests/test_gpu_bruss.py -k "3D_fused_step_kernel" > gpurun_out/sanitizer_racecheck.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/sanitizer_racecheck.log
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest -q -p no:cacheprovider \
  tests/test_gpu_bruss.py -k "3D_fused_step_kernel and shape2" > gpurun_out/sanitizer_synccheck.log 2>&1
echo "synccheck rc=$?" >> gpurun_out/sanitizer_synccheck.log
for f in gpurun_out/sanitizer_*.log; do tail -3 $f; done

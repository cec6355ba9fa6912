SUNBW_DEBUG=1 timeout 300 python -m pytest tests/test_gpu_fused_tol.py -q -p no:cacheprovider -k multirank -x 2>&1 | grep -E "sunbw|passed|failed" | head
SUNBW_PEER_HALO=0 timeout 300 python -m pytest tests/test_gpu_fused_tol.py -q -p no:cacheprovider -k multirank -x 2>&1 | tail -1
SUNBW_DEBUG=1 timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_fused_tol.py -q -p no:cacheprovider -k multirank -x 2>&1 | grep -v "^    " | head -40

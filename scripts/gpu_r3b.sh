TNB_GEMM_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -k "feed" -q -s 2>&1 | grep -E "k_gemm_fc|passed|failed" | sort | uniq -c | head -20

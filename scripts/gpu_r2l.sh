O=gpurun_out/${TAG:-r2l}; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -k "gemm_tc or group_kernels" -x -q > $O/pytest_tc.log 2>&1; echo "pytest tc exit $?"; tail -3 $O/pytest_tc.log
TNB_GEMM_DEBUG=1 timeout 300 python scripts/gemm_shape_bench.py 2>&1 | grep -v "^k_gemm R" | sort | uniq -c
TNB_GEMM_DEBUG=1 timeout 300 python scripts/gemm_shape_bench.py --cls "bcbaacaaxaxabab" 2>&1 | sort | uniq -c
for D in 8; do echo "dbg=$D"; TNB_TC_DBG=$D timeout 300 python scripts/gemm_shape_bench.py --kernels 4 --iters 1 2>&1 | grep "tc trace" | tail -45 | head -10; done

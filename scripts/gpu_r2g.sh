O=gpurun_out/${TAG:-r2g}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 300 python -m pytest tests/test_gpu_parity.py -k "gemm_tc" -x -q > $O/pytest_tc.log 2>&1; echo "pytest tc exit $?"; tail -1 $O/pytest_tc.log
for D in 0 1 2 3 4 7; do echo "dbg=$D"; TNB_TC_DBG=$D timeout 300 python scripts/gemm_shape_bench.py --kernels 4 2>&1 | tail -1; done
TNB_GEMM_DEBUG=1 python scripts/gemm_shape_bench.py --kernels 4 --iters 1 2>&1 | grep k_gemm_tc | head -1

O=gpurun_out/${TAG:-r2i}; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -k "gemm_tc or group_kernels" -x -q > $O/pytest_tc.log 2>&1; echo "pytest tc exit $?"; tail -1 $O/pytest_tc.log
for D in 0 4 7; do echo "dbg=$D"; TNB_TC_DBG=$D timeout 300 python scripts/gemm_shape_bench.py 2>&1 | tail -2; done
for D in 8 12; do echo "dbg=$D"; TNB_TC_DBG=$D timeout 300 python scripts/gemm_shape_bench.py --kernels 4 --iters 1 2>&1 | grep "tc trace" | tail -45 | head -8; done

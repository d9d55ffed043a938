timeout 300 python -m pytest tests/test_gpu_parity.py -k "gemm_tc" -x -q 2>&1 | tail -1
for D in 8; do echo "dbg=$D"; TNB_TC_DBG=$D timeout 300 python scripts/gemm_shape_bench.py --kernels 4 --iters 1 2>&1 | grep "tc trace" | tail -45 | head -6; done
timeout 300 python scripts/gemm_shape_bench.py 2>&1 | tail -2

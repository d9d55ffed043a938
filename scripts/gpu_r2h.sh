O=gpurun_out/${TAG:-r2h}; mkdir -p $O
for D in 8 12 15; do echo "dbg=$D"; TNB_TC_DBG=$D timeout 300 python scripts/gemm_shape_bench.py --kernels 4 --iters 1 2>&1 | grep "tc trace" | tail -45 | head -30; done

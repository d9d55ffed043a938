set -x; O=gpurun_out/${TAG:-r2d}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 300 python -m pytest tests/test_gpu_parity.py -k "gemm_tc or group_kernels" -x -q > $O/pytest_tc.log 2>&1; echo "pytest tc exit $?"; tail -3 $O/pytest_tc.log
timeout 300 python scripts/gemm_shape_bench.py > $O/shape.log 2>&1; echo "shape exit $?"; cat $O/shape.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 3 -c 1 -o $O/tc_top python scripts/gemm_shape_bench.py --kernels 4 --iters 1 > $O/ncu.log 2>&1; echo "ncu exit $?"; tail -3 $O/ncu.log

# k_gemm_hm: parity tests + timing on C5a's two GEMM shapes against k_gemm
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r4d
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "hm or group_kernels" -x > gpurun_out/r4d/pytest.log 2>&1; tail -15 gpurun_out/r4d/pytest.log
TNB_GEMM_DEBUG=1 timeout 300 python scripts/gemm_shape_bench.py --cls bcbaacaacacababcaabcaaaac --M 3 --kernels 1,5 > gpurun_out/r4d/shape_top.log 2>&1; tail -3 gpurun_out/r4d/shape_top.log
TNB_GEMM_DEBUG=1 timeout 300 python scripts/gemm_shape_bench.py --cls abccabcaabcbabaaacaaaaacba --M 3 --kernels 1,5 > gpurun_out/r4d/shape_fcprod.log 2>&1; tail -3 gpurun_out/r4d/shape_fcprod.log

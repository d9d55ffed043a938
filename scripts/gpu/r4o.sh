# k_gemm_hm tuning on C5a's top group: hoisted offsets / non-volatile mma; ring depth
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r4o; mkdir -p $O
for st in 3 2 4; do TNB_HM_STAGES=$st timeout 300 python scripts/gemm_shape_bench.py --cls bcbaacaacacababcaabcaaaac --M 3 --kernels 1,5 --iters 50 2>&1 | grep kernel | sed "s/^/S=$st /"; done | tee $O/shape_top.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "hm" > $O/pytest.log 2>&1; tail -1 $O/pytest.log

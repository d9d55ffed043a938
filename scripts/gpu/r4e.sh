# ncu of k_gemm_hm on C5a's top group shape
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r4e
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_hm -c 1 -o gpurun_out/r4e/hm_top python scripts/gemm_shape_bench.py --cls bcbaacaacacababcaabcaaaac --M 3 --kernels 5 --iters 2 > gpurun_out/r4e/ncu.log 2>&1
tail -2 gpurun_out/r4e/ncu.log

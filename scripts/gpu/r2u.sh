# ncu --set full of C5a's top k_gemm (op27, the 3rd M=3 launch of a slice) and the k_gemm_fc launch
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2u
timeout 300 python scripts/c5a_one_pass.py C5a 1 > gpurun_out/r2u/plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_gemm<3" --launch-skip 2 --launch-count 1 -o gpurun_out/r2u/gemm_top python scripts/c5a_one_pass.py C5a 1 > gpurun_out/r2u/ncu1.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_gemm_fc" --launch-count 1 -o gpurun_out/r2u/gemm_fc python scripts/c5a_one_pass.py C5a 1 > gpurun_out/r2u/ncu2.log 2>&1
tail -2 gpurun_out/r2u/ncu1.log gpurun_out/r2u/ncu2.log

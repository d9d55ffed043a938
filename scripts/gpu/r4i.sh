# ncu of k_fc_hm (C5a pair) and k_gemm_hm (top group)
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r4i
TNB_ONE_LANE=1 TNB_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_hm --launch-skip 2 -c 1 \
  -o gpurun_out/r4i/hm python scripts/c5a_one_pass.py C5a 1 > gpurun_out/r4i/ncu.log 2>&1
tail -2 gpurun_out/r4i/ncu.log

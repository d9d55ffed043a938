# ncu --set full of every k_gemm / k_gemm_fc launch of one C5a slice (prefix + slice 0), plus the step profile
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r4b
TNB_ONE_LANE=1 timeout 300 python scripts/step_profile.py --workload C5a > gpurun_out/r4b/steps.txt 2>&1
TNB_ONE_LANE=1 TNB_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm \
  -o gpurun_out/r4b/kgemm python scripts/c5a_one_pass.py C5a 1 > gpurun_out/r4b/ncu.log 2>&1
tail -2 gpurun_out/r4b/ncu.log

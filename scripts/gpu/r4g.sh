# per-launch times of one C5a slice with and without k_gemm_hm
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r4g
for v in 1 0; do TNB_GEMM_HM=$v TNB_ONE_LANE=1 timeout 300 python scripts/step_profile.py --workload C5a > gpurun_out/r4g/steps_hm$v.txt 2>&1; done
TNB_GEMM_DEBUG=1 TNB_ONE_LANE=1 TNB_GRAPH=0 timeout 300 python scripts/c5a_one_pass.py C5a 1 2>&1 | grep "k_gemm_hm R" > gpurun_out/r4g/hm_shapes.txt
head -30 gpurun_out/r4g/steps_hm1.txt

set -x; O=gpurun_out/${TAG:-r1c}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_gpu_parity.py -k "group_kernels" -x -q > $O/pytest_group.log 2>&1; echo "pytest group exit $?"; tail -15 $O/pytest_group.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench.log 2>&1; echo "bench exit $?"; tail -c 1200 $O/bench.log
TNB_NO_GEMM=1 timeout 600 python bench.py --no-cpu-baseline > $O/bench_nogemm.log 2>&1; echo "bench nogemm exit $?"; tail -c 300 $O/bench_nogemm.log
timeout 600 python scripts/step_profile.py --out $O/steps.json > $O/steps.log 2>&1; echo "steps exit $?"; head -25 $O/steps.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_gemm" -c 10 -o $O/prof_gemm python scripts/profile_c5a.py > $O/ncu_top.log 2>&1; echo "ncu top exit $?"

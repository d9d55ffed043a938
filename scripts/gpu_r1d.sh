set -x; O=gpurun_out/${TAG:-r1d}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench.log 2>&1; echo "bench exit $?"; tail -c 1200 $O/bench.log
timeout 600 python scripts/step_profile.py --out $O/steps.json > $O/steps.log 2>&1; echo "steps exit $?"; head -25 $O/steps.log
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_gemm<3" -c 3 -o $O/prof_gemm3 python scripts/profile_c5a.py > $O/ncu_top.log 2>&1; echo "ncu top exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_group_t<float2, unsigned int, 1, 1, 5" -c 1 -o $O/prof_group5 python scripts/profile_c5a.py > $O/ncu_g5.log 2>&1; echo "ncu g5 exit $?"

set -x; O=gpurun_out/${TAG:-r1j}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_gpu_parity.py -k "group_kernels or fused" -x -q > $O/pytest_group.log 2>&1; echo "pytest group exit $?"; tail -2 $O/pytest_group.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest_gpu.log
for L in 1 2 3 4; do TNB_LANES=$L timeout 600 python bench.py --no-cpu-baseline > $O/bench_l$L.log 2>&1; echo "bench L=$L exit $?"; python -c "import json;d=json.loads(open('$O/bench_l$L.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path'])"; done
timeout 600 python scripts/step_profile.py --out $O/steps.json > $O/steps.log 2>&1; echo "steps exit $?"; head -14 $O/steps.log
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_gemm<.int.3" -c 3 -o $O/prof_gemm3 python scripts/profile_c5a.py --records $O/recs.json > $O/ncu_top.log 2>&1; echo "ncu top exit $?"; tail -2 $O/ncu_top.log
python scripts/ncu_traffic.py --rep $O/prof_gemm3.ncu-rep --records $O/recs.json --kernel k_gemm --M 3 > $O/traffic.log 2>&1; cat $O/traffic.log
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_group_t<float2, unsigned int, .int.1, .int.1, .int.5" -c 1 -o $O/prof_group5 python scripts/profile_c5a.py > $O/ncu_g5.log 2>&1; echo "ncu g5 exit $?"

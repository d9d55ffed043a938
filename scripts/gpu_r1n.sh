set -x; O=gpurun_out/${TAG:-r1n}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench exit $?"; python -c "import json;d=json.loads(open('$O/bench.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path'],r['families'])"
TNB_LANES=1 timeout 900 python bench.py --no-cpu-baseline > $O/bench_1lane.log 2>&1; echo "bench 1lane exit $?"; python -c "import json;d=json.loads(open('$O/bench_1lane.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path'])"
timeout 600 python scripts/step_profile.py --out $O/steps.json > $O/steps.log 2>&1; echo "steps exit $?"; head -16 $O/steps.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu launches exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_gemm<.int.3" -c 4 -o $O/prof_gemm3 python scripts/profile_c5a.py --records $O/recs.json > $O/ncu_top.log 2>&1; echo "ncu top exit $?"; tail -2 $O/ncu_top.log
python scripts/ncu_traffic.py --rep $O/prof_gemm3.ncu-rep --records $O/recs.json --kernel k_gemm --M 3 > $O/traffic.log 2>&1; cat $O/traffic.log

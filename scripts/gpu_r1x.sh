set -x; O=gpurun_out/${TAG:-r1x}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 300 python -m pytest tests/test_gpu_parity.py -k "group_kernels" -x -q > $O/pytest_group.log 2>&1; echo "pytest group exit $?"; tail -15 $O/pytest_group.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 $O/pytest_gpu.log
for W in 1 0; do TNB_GEMM_WS=$W timeout 900 python bench.py --no-cpu-baseline > $O/bench_ws$W.log 2>&1; echo "bench WS=$W exit $?"; python -c "import json;d=json.loads(open('$O/bench_ws$W.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path']['frac'],{k:(round(v['ms_share_of_step'],3),round(v['GBps'])) for k,v in r['families'].items()},d['clocks'])"; done
timeout 600 python scripts/step_profile.py --out $O/steps.json > $O/steps.log 2>&1; head -6 $O/steps.log
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_gemm_ws<.int.3" -c 4 -o $O/prof_ws3 python scripts/profile_c5a.py --records $O/recs.json > $O/ncu_top.log 2>&1; echo "ncu exit $?"
python scripts/ncu_traffic.py --rep $O/prof_ws3.ncu-rep --records $O/recs.json --kernel k_gemm --M 3 > $O/traffic.log 2>&1; cat $O/traffic.log

set -x; O=gpurun_out/${TAG:-r1q}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest_gpu.log
for R3 in 1 0; do TNB_GEMM_RA3=$R3 timeout 900 python bench.py --no-cpu-baseline > $O/bench_ra$R3.log 2>&1; echo "bench RA3=$R3 exit $?"; python -c "import json;d=json.loads(open('$O/bench_ra$R3.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path']['frac'],{k:(round(v['ms_share_of_step'],3),round(v['GBps'])) for k,v in r['families'].items()})"; done
timeout 600 python scripts/step_profile.py --out $O/steps.json > $O/steps.log 2>&1; head -8 $O/steps.log
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_gemm<.int.3" -c 4 -o $O/prof_gemm3 python scripts/profile_c5a.py --records $O/recs.json > $O/ncu_top.log 2>&1; echo "ncu top exit $?"
python scripts/ncu_traffic.py --rep $O/prof_gemm3.ncu-rep --records $O/recs.json --kernel k_gemm --M 3 > $O/traffic.log 2>&1; cat $O/traffic.log

set -x; O=gpurun_out/${TAG:-r2c}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 300 python -m pytest tests/test_gpu_parity.py -k "gemm_tc or group_kernels" -x -q > $O/pytest_tc.log 2>&1; echo "pytest tc exit $?"; tail -3 $O/pytest_tc.log
for TC in 1; do TNB_GEMM_TC=$TC timeout 900 python bench.py --no-cpu-baseline > $O/bench_tc$TC.log 2>&1; echo "bench TC=$TC exit $?"; python -c "import json;d=json.loads(open('$O/bench_tc$TC.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path']['frac'],{k:(round(v['ms_share_of_step'],3),round(v['GBps'])) for k,v in r['families'].items()},d['clocks'])"; done
timeout 600 python scripts/step_profile.py --out $O/steps.json > $O/steps.log 2>&1; head -12 $O/steps.log

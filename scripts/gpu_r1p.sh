set -x; O=gpurun_out/${TAG:-r1p}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
for WB in 2 3; do TNB_GEMM_WB=$WB timeout 600 python -m pytest tests/test_gpu_parity.py -k "group_kernels or fused or batch" -x -q > $O/pytest_wb$WB.log 2>&1; echo "pytest WB=$WB exit $?"; tail -2 $O/pytest_wb$WB.log; done
for WB in 2 3; do TNB_GEMM_WB=$WB timeout 900 python bench.py --no-cpu-baseline > $O/bench_wb$WB.log 2>&1; echo "bench WB=$WB exit $?"; python -c "import json;d=json.loads(open('$O/bench_wb$WB.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path']['frac'],{k:(round(v['ms_share_of_step'],3),round(v['GBps'])) for k,v in r['families'].items()})"; done
TNB_GEMM_WB=2 timeout 600 python scripts/step_profile.py --out $O/steps_wb2.json > $O/steps_wb2.log 2>&1; head -8 $O/steps_wb2.log

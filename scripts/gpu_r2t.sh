O=gpurun_out/${TAG:-r2t}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -k "chain or fused or feed or amplitude" -x -q 2>&1 | tail -1
for MM in 1 2; do TNB_GEMM_MIN_M=$MM timeout 900 python bench.py --no-cpu-baseline > $O/bench_mm$MM.log 2>&1; echo "bench MIN_M=$MM exit $?"; python -c "import json;d=json.loads(open('$O/bench_mm$MM.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path']['frac'],{k:(round(v['ms_share_of_step'],3),round(v['GBps'])) for k,v in r['families'].items()})"; done
TNB_GEMM_MIN_M=2 timeout 600 python scripts/step_profile.py --out $O/steps.json > $O/steps.log 2>&1; head -16 $O/steps.log

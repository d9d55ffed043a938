O=gpurun_out/${TAG:-r2o}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -k "feed or fused_groups" -x -q > $O/pytest_fc.log 2>&1; echo "pytest fc exit $?"; tail -15 $O/pytest_fc.log
TNB_GEMM_DEBUG=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep k_gemm_fc | sort | uniq -c
for F in 0 1; do TNB_NO_FEED=$F timeout 900 python bench.py --no-cpu-baseline > $O/bench_nofeed$F.log 2>&1; echo "bench NO_FEED=$F exit $?"; python -c "import json;d=json.loads(open('$O/bench_nofeed$F.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path']['frac'],{k:(round(v['ms_share_of_step'],3),round(v['GBps'])) for k,v in r['families'].items()},d['clocks'])"; done
timeout 600 python scripts/step_profile.py --out $O/steps.json > $O/steps.log 2>&1; head -8 $O/steps.log

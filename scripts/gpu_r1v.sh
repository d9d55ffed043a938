set -x; O=gpurun_out/${TAG:-r1v}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 $O/pytest_gpu.log
for C in 0 1; do TNB_GEMM_CONTIG=$C timeout 900 python bench.py --no-cpu-baseline > $O/bench_c$C.log 2>&1; echo "bench CONTIG=$C exit $?"; python -c "import json;d=json.loads(open('$O/bench_c$C.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path']['frac'],{k:(round(v['ms_share_of_step'],3),round(v['GBps'])) for k,v in r['families'].items()},d['clocks'])"; done
TNB_GEMM_CONTIG=1 timeout 600 python scripts/step_profile.py --out $O/steps_c1.json > $O/steps_c1.log 2>&1; head -6 $O/steps_c1.log

O=gpurun_out/${TAG:-r2n}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.log 2>&1; echo "bench exit $?"; python -c "import json;d=json.loads(open('$O/bench.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path']['frac'],{k:(round(v['ms_share_of_step'],3),round(v['GBps'])) for k,v in r['families'].items()},d['clocks'])"

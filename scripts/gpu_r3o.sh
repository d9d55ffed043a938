O=gpurun_out/r3o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -k "amplitude or interpreter or energy" -q 2>&1 | tail -1
timeout 900 python bench.py --workload C2 --no-cpu-baseline --steps 20 > $O/c2.log 2>&1; python -c "import json;d=json.loads(open('$O/c2.log').read().strip().splitlines()[-1]);print('C2', round(d['value'],2), d['ms_per_step'], {k:(round(v['ms_share_of_step'],3), round(v['GBps']), v['launches']) for k,v in d['roofline']['families'].items()}, d['gpu_launches'])"
timeout 900 python tests/run_configs.py --only C2 --out $O/cfg_C2.json > $O/cfg_C2.log 2>&1; python -c "import json;d=json.loads(open('$O/cfg_C2.log').read().strip().splitlines()[-1]);print(d['ms_per_contraction_c64'], d['parity'])"

O=gpurun_out/r3n; mkdir -p $O
timeout 900 python bench.py --workload C2 --no-cpu-baseline --steps 20 > $O/c2.log 2>&1; python -c "import json;d=json.loads(open('$O/c2.log').read().strip().splitlines()[-1]);print('C2', round(d['value'],2), d['ms_per_step'], {k:(round(v['ms_share_of_step'],3), round(v['GBps']), v['launches']) for k,v in d['roofline']['families'].items()}, d['gpu_launches'])"
timeout 600 python scripts/step_profile.py --workload C2 --out $O/steps.json > $O/steps.log 2>&1; head -14 $O/steps.log

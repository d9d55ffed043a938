O=gpurun_out/r3c; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -k "feed" -q 2>&1 | tail -1
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline --steps 20 > $O/b$i.log 2>&1; python -c "import json;d=json.loads(open('$O/b$i.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['value'],2),{k:(round(v['ms_share_of_step'],3),round(v['GBps'])) for k,v in r['families'].items()})"; done
timeout 600 python scripts/step_profile.py --out $O/steps.json > $O/steps.log 2>&1; head -3 $O/steps.log

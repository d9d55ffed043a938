O=gpurun_out/r3l; mkdir -p $O
for L in 4 8; do TNB_LANES=$L timeout 900 python bench.py --workload C4b --no-cpu-baseline --steps 10 > $O/c4b_$L.log 2>&1; python -c "import json;d=json.loads(open('$O/c4b_$L.log').read().strip().splitlines()[-1]);print('C4b lanes $L', round(d['value'],2), d['config']['plan']['workspace_GB'])"; done

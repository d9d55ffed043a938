O=gpurun_out/r3a; mkdir -p $O
for I in 0 1 2 3; do TNB_RECIPE_INDEX=$I timeout 900 python bench.py --no-cpu-baseline --steps 10 > $O/b$I.log 2>&1; python -c "import json;d=json.loads(open('$O/b$I.log').read().strip().splitlines()[-1]);print('recipe $I', d['config']['plan']['k'], d['config']['plan']['width'], round(d['value'],2), round(d['config']['algorithmic_GB_per_step'],1))"; done

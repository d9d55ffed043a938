O=gpurun_out/r2x; mkdir -p $O
for v in 0 32 0; do TNB_CHAIN_NV=$v timeout 900 python tests/run_configs.py --only C4b --out $O/c4b_$v.json > $O/c4b_$v.log 2>&1; python -c "import json;d=json.loads(open('$O/c4b_$v.log').read().strip().splitlines()[-1]);print('NV=$v', d['ms_per_contraction_c64'])"; done
TNB_CHAIN_NV=32 timeout 900 python bench.py --no-cpu-baseline --steps 10 > $O/b32.log 2>&1; python -c "import json;d=json.loads(open('$O/b32.log').read().strip().splitlines()[-1]);print('bench NV=32', d['value'])"

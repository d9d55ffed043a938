O=gpurun_out/r2y; mkdir -p $O
for L in 3 4 5 6; do TNB_LANES=$L timeout 900 python bench.py --no-cpu-baseline --steps 10 > $O/bl$L.log 2>&1; python -c "import json;d=json.loads(open('$O/bl$L.log').read().strip().splitlines()[-1]);print('lanes $L', round(d['value'],2), d['clocks']['reasons'])"; done
for S in 2 4; do TNB_GEMM_STAGES=$S timeout 900 python bench.py --no-cpu-baseline --steps 10 > $O/bs$S.log 2>&1; python -c "import json;d=json.loads(open('$O/bs$S.log').read().strip().splitlines()[-1]);print('stages $S', round(d['value'],2))"; done

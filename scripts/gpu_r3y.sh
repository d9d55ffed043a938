O=gpurun_out/r3y; mkdir -p $O
for E in "X=0" "TNB_GEMM_RA3=1" "TNB_GEMM_STAGES=4" "TNB_GEMM_STAGES=2" "TNB_GEMM_WS=1" "TNB_LANES=6" "X=1"; do env $E timeout 900 python bench.py --no-cpu-baseline --steps 20 > $O/b.log 2>&1; python -c "import json;d=json.loads(open('$O/b.log').read().strip().splitlines()[-1]);print('$E', round(d['value'],2))"; done

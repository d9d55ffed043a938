O=gpurun_out/r3z; mkdir -p $O
TNB_FC_WB=2 timeout 900 python -m pytest tests/test_gpu_parity.py -k "feed or fused or c5a or lanes" -q 2>&1 | tail -1
for E in "TNB_FC_WB=2" "X=0" "TNB_FC_WB=2" "X=0"; do env $E timeout 900 python bench.py --no-cpu-baseline --steps 30 > $O/b.log 2>&1; python -c "import json;d=json.loads(open('$O/b.log').read().strip().splitlines()[-1]);print('C5a $E', round(d['value'],2))"; done
for E in "TNB_FC_WB=2" "X=0"; do env $E timeout 900 python bench.py --workload C4b --no-cpu-baseline --steps 20 > $O/c.log 2>&1; python -c "import json;d=json.loads(open('$O/c.log').read().strip().splitlines()[-1]);print('C4b $E', round(d['value'],2))"; done

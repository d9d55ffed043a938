O=gpurun_out/r3x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -k "group_kernels or fused or feed or c5a or amplitude" -q 2>&1 | tail -1
for W in C5a C5a C4b; do timeout 900 python bench.py --workload $W --no-cpu-baseline --steps 30 > $O/b.log 2>&1; python -c "import json;d=json.loads(open('$O/b.log').read().strip().splitlines()[-1]);print('$W', round(d['value'],2))"; done
TNB_GEMM_WB=3 timeout 900 python bench.py --workload C4b --no-cpu-baseline --steps 30 > $O/b.log 2>&1; python -c "import json;d=json.loads(open('$O/b.log').read().strip().splitlines()[-1]);print('C4b WB=3', round(d['value'],2))"

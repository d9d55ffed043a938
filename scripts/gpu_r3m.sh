O=gpurun_out/r3m; mkdir -p $O
for W in C5a C4b; do timeout 900 python bench.py --workload $W --no-cpu-baseline --steps 20 > $O/$W.log 2>&1; python -c "import json;d=json.loads(open('$O/$W.log').read().strip().splitlines()[-1]);print('$W', round(d['value'],2), d['roofline'].get('concurrent_slice_lanes'), d['clocks'])"; done
timeout 900 python -m pytest tests/test_gpu_parity.py -k "lanes or c5a or feed" -q 2>&1 | tail -1

# confirm the k_gemm_fc revert: per-launch time and bench
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r4m; mkdir -p $O
TNB_ONE_LANE=1 timeout 300 python scripts/step_profile.py --workload C5a > $O/steps.txt 2>&1; head -2 $O/steps.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; python -c "
import json; d=json.load(open('$O/bench.json')); r=d['roofline']; print('C5a', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['frac'])"

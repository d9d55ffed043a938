# C5a: fused pair (k_gemm_fc) vs unfused (producer on k_gemm_hm + consumer) now that k_gemm_hm exists
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r4p; mkdir -p $O
for v in 0 1; do TNB_NO_FC=$v TNB_ONE_LANE=1 timeout 300 python scripts/step_profile.py --workload C5a > $O/steps_nofc$v.txt 2>&1; head -4 $O/steps_nofc$v.txt; done
for v in 0 1; do TNB_NO_FC=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_nofc$v.json 2> $O/bench_nofc$v.err; python -c "
import json; d=json.load(open('$O/bench_nofc$v.json')); r=d['roofline']; print('NO_FC=$v C5a', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['frac'])"; done

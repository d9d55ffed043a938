# DFMA vs DMMA rate (c128 justification); C5r (paper-replica plan, 2^30 steps) with / without k_gemm_hm
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r4n; mkdir -p $O
./scripts/probe/mma_rate.bin > $O/mma_rate.txt 2>&1; grep -E "dfma|f64" $O/mma_rate.txt
for v in 1 0; do TNB_GEMM_HM=$v TNB_ONE_LANE=1 timeout 600 python scripts/step_profile.py --workload C5r > $O/steps_C5r_hm$v.txt 2>&1; head -6 $O/steps_C5r_hm$v.txt; done
for v in 1 0; do TNB_GEMM_HM=$v timeout 900 python bench.py --workload C5r --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_C5r_hm$v.json 2> $O/bench_C5r_hm$v.err; python -c "
import json; d=json.load(open('$O/bench_C5r_hm$v.json')); r=d['roofline']; print('HM=$v C5r', d['value'], d['ms_per_step'], r['kernel'], r['bound'], r['frac'])"; done

# does k_fc_tc win on any other workload's pair shapes?  (C5r6, C4b, C5r, C2)
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2w
for w in C5r6 C4b C2; do
for v in 1 0; do
TNB_FC_TC=$v TNB_GEMM_DEBUG=1 timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2w/bench_${w}_tc$v.json 2> gpurun_out/r2w/bench_${w}_tc$v.err
python -c "
import json; d=json.load(open('gpurun_out/r2w/bench_${w}_tc$v.json')); r=d['roofline']; print('$w TC=$v', d['value'], 'ms', d['ms_per_step'], json.dumps({k:(round(v['ms_share_of_step'],3), v['launches']) for k,v in r['families'].items()}))"
grep -a "k_fc_tc R=\|k_fc_tc declined" gpurun_out/r2w/bench_${w}_tc$v.err | sort | uniq -c | head -4
done
done

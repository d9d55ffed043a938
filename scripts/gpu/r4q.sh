# other workloads with the round-2 final kernels (HM on / off): C4b, C2, C5a c128
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r4q; mkdir -p $O
for w in C4b C2; do for v in 1 0; do TNB_GEMM_HM=$v timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_${w}_hm$v.json 2> $O/bench_${w}_hm$v.err; python -c "
import json; d=json.load(open('$O/bench_${w}_hm$v.json')); r=d['roofline']; print('$w HM=$v', round(d['value'],2), d['unit'], round(d['ms_per_step'],3), 'ms', r['kernel'], r['bound'], round(r['frac'],3))"; done; done
timeout 900 python bench.py --steps 10 --warmup 3 --dtype c128 --no-cpu-baseline > $O/bench_c128.json 2> $O/bench_c128.err; python -c "
import json; d=json.load(open('$O/bench_c128.json')); r=d['roofline']; print('C5a c128', d['value'], r['kernel'], r['bound'], r['frac'])"

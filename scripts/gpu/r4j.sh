# k_gemm_fc with / without the L2 prefetch of the next tile's X; C5a bench
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r4j
for v in 1 0; do TNB_FC_XPF=$v TNB_ONE_LANE=1 timeout 300 python scripts/step_profile.py --workload C5a > gpurun_out/r4j/steps_xpf$v.txt 2>&1; head -3 gpurun_out/r4j/steps_xpf$v.txt; done
for v in 1 0; do TNB_FC_XPF=$v timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r4j/bench_xpf$v.json 2> gpurun_out/r4j/bench_xpf$v.err; python -c "
import json; d=json.load(open('gpurun_out/r4j/bench_xpf$v.json')); r=d['roofline']; print('XPF=$v C5a', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['frac'], {k: (round(v['ms_share_of_step'],3), round(v['GBps'])) for k,v in r['families'].items()})"; done

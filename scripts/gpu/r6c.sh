# k_gemm_fc grid variants in the 16-lane step: whole blocks (default), split blocks, one CTA per SM
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r6c; mkdir -p $O
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$tag.json 2>> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench_$tag.json')); r=d['roofline']; print('$tag C5a', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), r['kernel'], round(r['frac'],3), round(r['avg_launch_ms']*1e3,1), 'us')"; }
run base TNB_FC_SPLIT=0
run s1c1 TNB_FC_SPLIT=1 TNB_FC_CPS=1
run s0c1 TNB_FC_SPLIT=0 TNB_FC_CPS=1
run s1l24 TNB_FC_SPLIT=1 TNB_LANES=24
run base2 TNB_FC_SPLIT=0
run s1c1b TNB_FC_SPLIT=1 TNB_FC_CPS=1

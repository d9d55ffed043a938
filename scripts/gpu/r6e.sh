# slice-lane stream priorities (TNB_LANE_PRIO 0 / 1 graded / 2 alternating), interleaved A/B on C5a and C4b
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r6e; mkdir -p $O
run() { tag=$1; wl=$2; shift; shift; env "$@" timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$tag.json 2>> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench_$tag.json')); print('$tag', round(d['value'],2), 'e2e', round(d['e2e']['value'],2))"; }
for rep in a b; do for m in 0 1 2; do run C5a_p${m}_$rep C5a TNB_LANE_PRIO=$m; done; done
run C5a_p1_nograph C5a TNB_LANE_PRIO=1 TNB_GRAPH=0
run C5a_p0_nograph C5a TNB_LANE_PRIO=0 TNB_GRAPH=0
for m in 0 1 2; do run C4b_p$m C4b TNB_LANE_PRIO=$m; done

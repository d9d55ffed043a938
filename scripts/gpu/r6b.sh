# k_gemm_fc split consumer blocks (balanced tile ranges): parity (GPU suite), per-launch time and bench A/B
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r6b; mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -x -k "feed or fc or C5a or c5a or C4b or slice" > $O/pytest_fc.log 2>&1; tail -2 $O/pytest_fc.log
for v in 1 0; do TNB_FC_SPLIT=$v timeout 300 python scripts/step_profile.py --workload C5a > $O/steps_split$v.txt 2>&1; head -2 $O/steps_split$v.txt; done
for v in 1 0 1 0; do TNB_FC_SPLIT=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_split$v.json 2>> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench_split$v.json')); r=d['roofline']; print('split $v C5a', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), r['kernel'], round(r['frac'],3), round(r['avg_launch_ms']*1e3,1), 'us')"; done
for v in 1 0; do TNB_FC_SPLIT=$v timeout 600 python bench.py --workload C4b --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C4b_split$v.json 2>> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench_C4b_split$v.json')); print('split $v C4b', round(d['value'],2), d['unit'])"; done
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log

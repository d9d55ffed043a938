# full GPU suite + smoke with k_gemm_hm64 in the c128 path
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r5c; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
for w in C4b C2; do timeout 600 python bench.py --workload $w --dtype c128 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_${w}_c128.json 2> $O/bench_${w}_c128.err; python -c "
import json; d=json.load(open('$O/bench_${w}_c128.json')); r=d['roofline']; print('$w c128', round(d['value'],2), d['unit'], r['kernel'], r['bound'], round(r['frac'],3))"; done
for w in C4b C2; do TNB_GEMM_HM64=0 timeout 600 python bench.py --workload $w --dtype c128 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_${w}_c128_off.json 2> /dev/null; python -c "
import json; d=json.load(open('$O/bench_${w}_c128_off.json')); r=d['roofline']; print('$w c128 HM64=0', round(d['value'],2), d['unit'], r['kernel'])"; done

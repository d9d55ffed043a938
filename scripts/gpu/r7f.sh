# final validation of the round (session 4): GPU suite, smoke, bench line (with cpu_baseline), the other
# workloads, ncu launch list of the bench, ncu --set full (with source counters) of the k_gemm_fc launch
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r7f; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench.json')); r=d['roofline']; print('C5a', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['bound'], r['frac'], r['unit'], d['gpu_launches'], d.get('cpu_baseline',{}).get('value'), d['clocks'])"
timeout 600 python bench.py --dtype c128 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c128.json 2>> $O/bench.err
for wl in C4b C2; do timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$wl.json 2>> $O/bench.err; python -c "
import json; d=json.load(open('$O/bench_$wl.json')); print('$wl', round(d['value'],2), d['unit'], round(d['ms_per_step'],4), 'ms')"; done
python -c "
import json; d=json.load(open('$O/bench_c128.json')); print('C5a c128', round(d['value'],2), 'e2e', round(d['e2e']['value'],2))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1; tail -1 $O/ncu_bench.log
TNB_GRAPH=0 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_gemm_fc --launch-count 1 -o $O/gemm_fc python scripts/c5a_one_pass.py C5a 1 > $O/ncu_fc.log 2>&1; tail -1 $O/ncu_fc.log
ncu -i $O/gemm_fc.ncu-rep > $O/ncu_full_gemm_fc.txt 2>&1
ncu -i $O/gemm_fc.ncu-rep --page raw --csv > $O/ncu_full_gemm_fc_raw.csv 2>&1
ncu -i $O/gemm_fc.ncu-rep --page source --csv > $O/ncu_gemm_fc_source.csv 2>&1

# validation of the session's default state: GPU suite, smoke, bench (with cpu_baseline), ncu launch
# lists (bench and one C5a slice with DRAM bytes), ncu --set full of k_gemm_hm / k_gemm_fc
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r4v; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench.json')); r=d['roofline']; print('C5a', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['bound'], r['frac'], r['unit'], d['gpu_launches'], d.get('cpu_baseline',{}).get('value'))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1; tail -1 $O/ncu_bench.log
TNB_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/c5a_slice_dram.csv python scripts/c5a_one_pass.py C5a 1 > $O/ncu_slice.log 2>&1; tail -1 $O/ncu_slice.log
TNB_GRAPH=0 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_gemm_hm -o $O/gemm_hm python scripts/c5a_one_pass.py C5a 1 > $O/ncu_hm.log 2>&1; tail -1 $O/ncu_hm.log
TNB_GRAPH=0 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_gemm_fc --launch-count 1 -o $O/gemm_fc python scripts/c5a_one_pass.py C5a 1 > $O/ncu_fc.log 2>&1; tail -1 $O/ncu_fc.log

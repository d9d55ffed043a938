# final profiles after the k_gemm default change: launch list, full captures, traffic, tests, bench
O=gpurun_out/final7; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench exit $?"; tail -1 $O/bench.log > $O/bench_c5a.jsonl
python -c "import json;d=json.loads(open('$O/bench_c5a.jsonl').read());r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],round(r['frac'],3),{k:(round(v['ms_share_of_step'],3),round(v['GBps'])) for k,v in r['families'].items()},d['clocks'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm<" -c 16 -o $O/ncu_full_kgemm python scripts/profile_c5a.py --records $O/recs.json > $O/ncu_kg.log 2>&1; echo "ncu kg exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_fc -s 1 -c 1 -o $O/ncu_full_kgemm_fc python scripts/profile_c5a.py --records $O/recs_fc.json > $O/ncu_fc.log 2>&1; echo "ncu fc exit $?"
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/smoke.log

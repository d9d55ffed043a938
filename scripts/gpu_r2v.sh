# round-1 final state: all configs (parity + timing), bench, ncu launch list, full captures + traffic
O=gpurun_out/final2; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
for c in C1 C3 C4b C5a C4a C2 C5b; do
  timeout 900 python tests/run_configs.py --only $c --out $O/cfg_$c.json > $O/cfg_$c.log 2> $O/cfg_$c.err; echo "$c exit $?"; tail -1 $O/cfg_$c.log
done
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench exit $?"; tail -1 $O/bench.log > $O/bench_c5a.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_fc -s 1 -c 1 -o $O/ncu_full_kgemm_fc python scripts/profile_c5a.py --records $O/recs.json > $O/ncu_fc.log 2>&1; echo "ncu fc exit $?"
python scripts/ncu_traffic.py --rep $O/ncu_full_kgemm_fc.ncu-rep --records $O/recs.json --kernel k_gemm_fc > $O/traffic_fc.txt 2>&1; cat $O/traffic_fc.txt | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_ws<.int.3" -c 4 -o $O/ncu_full_kgemm_ws3 python scripts/profile_c5a.py --records $O/recs2.json > $O/ncu_ws.log 2>&1; echo "ncu ws exit $?"
python scripts/ncu_traffic.py --rep $O/ncu_full_kgemm_ws3.ncu-rep --records $O/recs2.json --kernel k_gemm --M 3 > $O/traffic_ws.txt 2>&1; cat $O/traffic_ws.txt | tail -3
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -1 $O/pytest_gpu.log

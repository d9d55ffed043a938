# final validation of the committed state (round 1)
O=gpurun_out/final8; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench exit $?"; tail -1 $O/bench.log > $O/bench_c5a.jsonl
python -c "import json;d=json.loads(open('$O/bench_c5a.jsonl').read());r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],round(r['frac'],3),d['clocks'],d['gpu_launches'])"
for c in C5a C4b; do timeout 900 python tests/run_configs.py --only $c --out $O/cfg_$c.json > $O/cfg_$c.log 2> $O/cfg_$c.err; echo "$c exit $?"; done

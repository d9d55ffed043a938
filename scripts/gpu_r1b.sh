set -x; O=gpurun_out/${TAG:-r1b}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; nproc; lscpu | grep "Model name"
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench exit $?"; tail -c 1500 $O/bench.log
timeout 600 python scripts/step_profile.py --out $O/steps.json > $O/steps.log 2>&1; echo "steps exit $?"; head -25 $O/steps.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu launches exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_pair|k_group}" -c ${KCOUNT:-8} -o $O/prof_top python scripts/profile_c5a.py > $O/ncu_top.log 2>&1; echo "ncu top exit $?"

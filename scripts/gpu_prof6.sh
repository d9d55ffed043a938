set -x; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench default exit $?"
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_s1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches exit $?"
python scripts/profile_c5a.py > gpurun_out/prof_plain.log 2>&1; echo "plain exit $?"
SKIP=$(python scripts/profile_c5a.py --print-skip 173)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_bucket|k_group" -s $SKIP -c 3 -o gpurun_out/prof_top python scripts/profile_c5a.py > gpurun_out/ncu_top.log 2>&1; echo "ncu exit $?"

set -x; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
python scripts/profile_c5a.py > gpurun_out/prof_plain.log 2>&1; echo "plain exit $?"
SKIP=$(python scripts/profile_c5a.py --print-skip 164)
echo "skip=$SKIP"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_bucket -s $SKIP -c 4 -o gpurun_out/prof_c5a python scripts/profile_c5a.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
tail -5 gpurun_out/ncu_full.log
timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_s1.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches exit $?"
ls -la gpurun_out

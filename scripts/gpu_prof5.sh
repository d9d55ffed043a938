set -x; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
python scripts/profile_c5a.py > gpurun_out/prof_plain.log 2>&1; echo "plain exit $?"
SKIP=$(python scripts/profile_c5a.py --print-skip 173)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_bucket|k_group" -s $SKIP -c 1 -o gpurun_out/prof_g173 python scripts/profile_c5a.py > gpurun_out/ncu_g173.log 2>&1; echo "ncu exit $?"

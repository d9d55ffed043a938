set -x; O=gpurun_out/${TAG:-r1o}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench exit $?"; tail -c 3500 $O/bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1; echo "ref exit $?"; tail -c 1500 $O/bench_ref.log

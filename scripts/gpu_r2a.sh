set -x; O=gpurun_out/${TAG:-r2a}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 60 ./scripts/probe/tc_probe > $O/probe.log 2>&1; echo "probe exit $?"; cat $O/probe.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench exit $?"; tail -1 $O/bench.log | cut -c1-600

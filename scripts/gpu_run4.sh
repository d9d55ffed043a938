set -x; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/step_profile.py --out gpurun_out/steps_c5a.json > gpurun_out/steps.log 2>&1; echo "steps exit $?"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?"

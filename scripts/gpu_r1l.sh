set -x; O=gpurun_out/${TAG:-r1l}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_gpu_parity.py -k "batch or lanes" -x -q > $O/pytest_batch.log 2>&1; echo "pytest batch exit $?"; tail -15 $O/pytest_batch.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench exit $?"; python -c "import json;d=json.loads(open('$O/bench.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path'],d.get('cpu_baseline'))"
timeout 600 python scripts/step_profile.py --out $O/steps.json > $O/steps.log 2>&1; echo "steps exit $?"; head -12 $O/steps.log

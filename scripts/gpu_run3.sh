set -x; mkdir -p gpurun_out
timeout 600 python scripts/step_profile.py --out gpurun_out/steps_c5a.json > gpurun_out/steps.log 2>&1; echo "steps exit $?"; cat gpurun_out/steps.log

set -x; mkdir -p gpurun_out
for c in ${CFGS:-C1 C3 C4b C5a C4a C2 C5b}; do
  timeout 900 python tests/run_configs.py --only $c --out gpurun_out/cfg_$c.json > gpurun_out/cfg_$c.log 2> gpurun_out/cfg_$c.err; echo "$c exit $?"
  tail -2 gpurun_out/cfg_$c.err; free -g | head -2
done

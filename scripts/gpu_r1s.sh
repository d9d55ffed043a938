set -x; O=gpurun_out/${TAG:-r1s}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
free -g | head -2
timeout 2400 python tests/run_configs.py --out $O/configs.json > $O/configs.log 2> $O/configs.err; echo "configs exit $?"; tail -3 $O/configs.err
python - <<'PY'
import json
for r in json.load(open("gpurun_out/r1s/configs.json")):
    print({k: v for k, v in r.items() if k not in ("tried",)})
PY

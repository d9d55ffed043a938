set -x; O=gpurun_out/${TAG:-r1r}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
for L in 4 6 8; do TNB_LANES=$L timeout 900 python bench.py --no-cpu-baseline --steps 30 > $O/bench_l$L.log 2>&1; echo "bench L=$L exit $?"; python -c "import json;d=json.loads(open('$O/bench_l$L.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['path']['frac'],d['clocks'])"; done

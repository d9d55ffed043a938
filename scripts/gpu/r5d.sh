# k_gemm_hm64 size gate for c128 (TNB_HM64_MIN_R = 14 / 17 / 20 / 23)
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r5d; mkdir -p $O
for w in C5a C4b C2; do for m in 14 17 20 23; do TNB_HM64_MIN_R=$m timeout 600 python bench.py --workload $w --dtype c128 --steps 10 --warmup 3 --no-cpu-baseline > $O/b_${w}_$m.json 2>/dev/null; python -c "
import json; d=json.load(open('$O/b_${w}_$m.json')); print('$w c128 MIN_R=$m', round(d['value'],2))"; done; done

O=gpurun_out/r3q; mkdir -p $O
for S in 1 0; do TNB_FC_SHRINK=$S timeout 900 python bench.py --workload C4b --no-cpu-baseline --steps 20 > $O/c4b_$S.log 2>&1; python -c "import json;d=json.loads(open('$O/c4b_$S.log').read().strip().splitlines()[-1]);print('C4b shrink $S', round(d['value'],2), {k:(round(v['ms_share_of_step'],3), round(v['GBps'])) for k,v in d['roofline']['families'].items()})"; done
timeout 900 python bench.py --no-cpu-baseline --steps 10 > $O/c5a.log 2>&1; python -c "import json;d=json.loads(open('$O/c5a.log').read().strip().splitlines()[-1]);print('C5a', round(d['value'],2))"
timeout 900 python -m pytest tests/test_gpu_parity.py -k "feed or fused or multi_round" -q 2>&1 | tail -1
TNB_GEMM_DEBUG=1 timeout 600 python bench.py --workload C4b --no-cpu-baseline --steps 3 --warmup 3 2>&1 | grep "k_gemm_fc R" | sort | uniq -c

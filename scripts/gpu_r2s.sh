O=gpurun_out/${TAG:-r2s}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -k "feed or fused_groups" -x -q 2>&1 | tail -1
for R in 2 1; do TNB_FC_RBB=$R timeout 900 python bench.py --no-cpu-baseline > $O/bench_rbb$R.log 2>&1; echo "bench RBB=$R exit $?"; python -c "import json;d=json.loads(open('$O/bench_rbb$R.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path']['frac'],{k:(round(v['ms_share_of_step'],3),round(v['GBps'])) for k,v in r['families'].items()})"; done

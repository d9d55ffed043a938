O=gpurun_out/${TAG:-r2k}; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -k "gemm_tc or group_kernels" -x -q > $O/pytest_tc.log 2>&1; echo "pytest tc exit $?"; tail -1 $O/pytest_tc.log
TNB_GEMM_DEBUG=1 timeout 300 python scripts/gemm_shape_bench.py 2>&1 | grep -v "^k_gemm R" | sort | uniq -c
TNB_GEMM_DEBUG=1 timeout 300 python scripts/gemm_shape_bench.py --cls "bcbaacaaxaxabab" 2>&1 | tail -3
for D in 8; do echo "dbg=$D"; TNB_TC_DBG=$D timeout 300 python scripts/gemm_shape_bench.py --kernels 4 --iters 1 2>&1 | grep "tc trace" | tail -45 | head -8; done
TNB_GEMM_DEBUG=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep k_gemm_tc | sort | uniq -c
timeout 900 python bench.py --no-cpu-baseline > $O/bench.log 2>&1; echo "bench exit $?"; python -c "import json;d=json.loads(open('$O/bench.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path']['frac'],{k:(round(v['ms_share_of_step'],3),round(v['GBps'])) for k,v in r['families'].items()},d['clocks'])"

set -x; O=gpurun_out/${TAG:-r2b}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 300 python -m pytest tests/test_gpu_parity.py -k "gemm_tc" -x -q > $O/pytest_tc.log 2>&1; echo "pytest tc exit $?"; tail -25 $O/pytest_tc.log
timeout 300 python -m pytest tests/test_gpu_parity.py -k "group_kernels" -x -q > $O/pytest_group.log 2>&1; echo "pytest group exit $?"; tail -3 $O/pytest_group.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest_gpu.log
TNB_GEMM_DEBUG=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_dbg.log 2> $O/bench_dbg.err; echo "bench dbg exit $?"; sort $O/bench_dbg.err | uniq -c | sort -rn | head -30
for TC in 1 0; do TNB_GEMM_TC=$TC timeout 900 python bench.py --no-cpu-baseline > $O/bench_tc$TC.log 2>&1; echo "bench TC=$TC exit $?"; python -c "import json;d=json.loads(open('$O/bench_tc$TC.log').read().strip().splitlines()[-1]);r=d['roofline'];print(d['value'],d['e2e']['value'],r['kernel'],r['frac'],r['path']['frac'],{k:(round(v['ms_share_of_step'],3),round(v['GBps'])) for k,v in r['families'].items()},d['clocks'])"; done

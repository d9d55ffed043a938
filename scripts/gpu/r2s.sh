# k_gemm_fc X-first traversal A/B, DRAM of the fused launch, c128 bench line
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2s
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "feed or c5a or lanes" > gpurun_out/r2s/pytest.log 2>&1; tail -1 gpurun_out/r2s/pytest.log
for v in 1 0; do
TNB_FC_XFIRST=$v timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2s/bench_xf$v.json 2> gpurun_out/r2s/bench_xf$v.err
python -c "
import json; d=json.load(open('gpurun_out/r2s/bench_xf$v.json')); r=d['roofline']; print('XFIRST=$v VALUE', d['value'], 'e2e', d['e2e']['value']); print(json.dumps(r['families']))"
done
timeout 900 python bench.py --steps 10 --warmup 3 --dtype c128 --no-cpu-baseline > gpurun_out/r2s/bench_c128.json 2> gpurun_out/r2s/bench_c128.err
python -c "
import json; d=json.load(open('gpurun_out/r2s/bench_c128.json')); r=d['roofline']; print('C128 VALUE', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['frac'])"
timeout 300 python scripts/c5a_one_pass.py C5a 1 > gpurun_out/r2s/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2s/c5a_slice_dram.csv python scripts/c5a_one_pass.py C5a 1 > gpurun_out/r2s/ncu.log 2>&1
tail -1 gpurun_out/r2s/ncu.log

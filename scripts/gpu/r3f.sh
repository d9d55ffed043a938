# k_gemm_fc with the consumer factors X staged in shared memory one tile ahead (XS): geometry,
# parity (full -m gpu suite), bench XS on / off, ncu --set full of the XS launch
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r3f
TNB_GEMM_DEBUG=1 TNB_GRAPH=0 timeout 300 python scripts/c5a_one_pass.py C5a 1 2>&1 | grep "k_gemm_fc R=" | sort | uniq -c
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r3f/pytest_gpu.log 2>&1; tail -2 gpurun_out/r3f/pytest_gpu.log
for v in 1 0 1; do
TNB_FC_XS=$v timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3f/bench_xs$v.json 2> gpurun_out/r3f/bench_xs$v.err
python -c "
import json; d=json.load(open('gpurun_out/r3f/bench_xs$v.json')); f=d['roofline']['families']; print('XS=$v', d['value'], 'e2e', d['e2e']['value'], {k:round(v['ms_share_of_step'],3) for k,v in f.items()})"
done
timeout 300 python scripts/c5a_one_pass.py C5a 1 > gpurun_out/r3f/plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_gemm_fc" --launch-count 1 -o gpurun_out/r3f/gemm_fc_xs python scripts/c5a_one_pass.py C5a 1 > gpurun_out/r3f/ncu.log 2>&1
tail -2 gpurun_out/r3f/ncu.log

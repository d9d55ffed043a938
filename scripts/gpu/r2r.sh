# per-step profiles (C5a, C5r, C5r6), chain threshold A/B, per-launch DRAM bytes of one C5r slice
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2r
for w in C5a C5r C5r6; do
timeout 600 python scripts/step_profile.py --workload $w --out gpurun_out/r2r/steps_$w.json > gpurun_out/r2r/steps_$w.txt 2>&1
head -14 gpurun_out/r2r/steps_$w.txt
done
for v in 15 0; do
TNB_RUN_CHAIN_MIN=$v timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2r/bench_chain$v.json 2> gpurun_out/r2r/bench_chain$v.err
python -c "
import json; d=json.load(open('gpurun_out/r2r/bench_chain$v.json')); r=d['roofline']; print('CHAINMIN=$v VALUE', d['value'], 'e2e', d['e2e']['value'], d['gpu_launches']); print(json.dumps(r['families']))"
done
timeout 600 python scripts/c5a_one_pass.py C5r 1 > gpurun_out/r2r/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2r/c5r_slice_dram.csv python scripts/c5a_one_pass.py C5r 1 > gpurun_out/r2r/ncu.log 2>&1
tail -2 gpurun_out/r2r/ncu.log

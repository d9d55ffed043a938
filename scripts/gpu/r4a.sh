# round-2 session 2: restored-state check (bench C5a) + shapes of the C5a plan's GEMM groups
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r4a
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r4a/bench.json 2> gpurun_out/r4a/bench.err
python -c "
import json; d=json.load(open('gpurun_out/r4a/bench.json')); r=d['roofline']; print('C5a', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['frac'], d['gpu_launches'])"
TNB_GEMM_DEBUG=1 TNB_ONE_LANE=1 TNB_GRAPH=0 timeout 300 python scripts/c5a_one_pass.py C5a 1 > gpurun_out/r4a/shapes.log 2>&1
TNB_ONE_LANE=1 timeout 300 python scripts/step_profile.py C5a > gpurun_out/r4a/steps.txt 2>&1
tail -3 gpurun_out/r4a/shapes.log

# round 2: config parity tests, full gpu suite, bench with the all-core oracle baseline, the
# reference arm, and the 8-rank functional multi-rank line (gloo, one GPU: not a measurement)
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2b
timeout 1800 python -m pytest tests/test_gpu_configs.py -x -q -m gpu --durations=15 > gpurun_out/r2b/pytest_configs.log 2>&1
tail -25 gpurun_out/r2b/pytest_configs.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err
tail -c 1500 gpurun_out/r2b/bench.json
TNB_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 8 --steps 5 --warmup 3 > gpurun_out/r2b/bench_gloo8.json 2> gpurun_out/r2b/bench_gloo8.err
tail -c 800 gpurun_out/r2b/bench_gloo8.json; tail -5 gpurun_out/r2b/bench_gloo8.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2b/ref.json 2> gpurun_out/r2b/ref.err
cat gpurun_out/r2b/ref.json; tail -3 gpurun_out/r2b/ref.err

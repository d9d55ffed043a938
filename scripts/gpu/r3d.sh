# energy: shared-memory-resident cones (k_cone_smem) vs the L2 path; energy parity tests; oracle small timings
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r3d
for v in 1 0; do echo "CONE_SMEM=$v"; TNB_CONE_SMEM=$v timeout 600 python scripts/energy_timing.py; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "energy" > gpurun_out/r3d/pytest_energy.log 2>&1; tail -1 gpurun_out/r3d/pytest_energy.log
timeout 900 python scripts/oracle_small_timing.py --out gpurun_out/r3d/oracle_timing.json

# compute-sanitizer racecheck (shared-memory hazards) on the smoke plans (one tool per call)
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2q
timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2q/racecheck.log 2>&1
echo "racecheck rc=$?"; tail -5 gpurun_out/r2q/racecheck.log

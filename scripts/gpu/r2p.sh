# compute-sanitizer memcheck on the smoke plans (one tool per call)
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2p
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p/memcheck.log 2>&1
echo "memcheck rc=$?"; tail -5 gpurun_out/r2p/memcheck.log

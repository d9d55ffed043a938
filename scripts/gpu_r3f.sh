O=gpurun_out/r3f; mkdir -p $O
timeout 1200 python tests/run_configs.py --only C5b --out $O/cfg_C5b.json > $O/cfg_C5b.log 2> $O/cfg_C5b.err; echo "C5b exit $?"; tail -1 $O/cfg_C5b.log

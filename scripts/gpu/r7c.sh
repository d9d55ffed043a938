# ncu --set full with source counters of the k_gemm_fc launch (FC_U1=1 default): per-instruction executed counts
O=gpurun_out/r7c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python scripts/c5a_one_pass.py C5a 1 > $O/plain.log 2>&1; tail -1 $O/plain.log
TNB_GRAPH=0 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_gemm_fc --launch-count 1 -o $O/gemm_fc python scripts/c5a_one_pass.py C5a 1 > $O/ncu_fc.log 2>&1; tail -1 $O/ncu_fc.log
ncu -i $O/gemm_fc.ncu-rep > $O/ncu_full_gemm_fc.txt 2>&1
ncu -i $O/gemm_fc.ncu-rep --page raw --csv > $O/ncu_full_gemm_fc_raw.csv 2>&1
ncu -i $O/gemm_fc.ncu-rep --page source --csv > $O/ncu_gemm_fc_source.csv 2>&1
ls -la $O

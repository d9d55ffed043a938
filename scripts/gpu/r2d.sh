# round 2: ncu of the first k_fc_tc launch (C5a), source-level
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2d
TNB_FC_TC=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fc_tc -c 1 -o gpurun_out/r2d/fctc python scripts/c5a_one_pass.py > gpurun_out/r2d/ncu.log 2>&1
tail -3 gpurun_out/r2d/ncu.log

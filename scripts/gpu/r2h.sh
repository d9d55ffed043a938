python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2h
TNB_FC_TC=1 TNB_FT_TRACE=1 timeout 300 python scripts/c5a_one_pass.py C5a 3 2>&1 | grep -a "k_fc_tc" | head -5

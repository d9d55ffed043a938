# k_fc_hm diagnostics: pipeline only (no MMA / no consumer math) vs full, contiguous vs default tile
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r4r; mkdir -p $O
for d in 0 1 2 3; do TNB_FC_HM=1 TNB_HM_DBG=$d TNB_ONE_LANE=1 timeout 300 python scripts/step_profile.py --workload C5a 2>&1 | grep "176-183" | sed "s/^/DBG=$d /"; done | tee $O/dbg.txt

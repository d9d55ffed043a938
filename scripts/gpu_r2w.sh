O=gpurun_out/final2; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_ws|k_gemm<" -c 16 -o $O/ncu_full_kgemm python scripts/profile_c5a.py --records $O/recs3.json > $O/ncu_ws.log 2>&1; echo "ncu ws exit $?"
python scripts/ncu_traffic.py --rep $O/ncu_full_kgemm.ncu-rep --records $O/recs3.json --kernel k_gemm > $O/traffic_ws.txt 2>&1; cat $O/traffic_ws.txt | tail -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2

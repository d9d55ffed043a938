O=gpurun_out/${TAG:-r2r}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_fc -s 1 -c 1 -o $O/fc python scripts/profile_c5a.py > $O/ncu.log 2>&1; echo "ncu exit $?"; tail -2 $O/ncu.log

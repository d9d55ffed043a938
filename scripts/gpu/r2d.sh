# round 2: ncu of the first k_fc_tc launch (C5a), source-level
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2d
cat > /tmp/one.py <<'PY'
import bench, torch, paper_2012_02430_b200 as T
plan,g,ga,be,meta=bench.build_workload_plan('C5a')
p=torch.zeros(2*plan.n_slices,dtype=torch.float64,device='cuda')
ws=plan.workspace(T.TN_C64, batch=1)
T._binding.tn_contract_sliced(plan.handle, T.TN_C64, ga, be, 0, 2, ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream, p.data_ptr())
torch.cuda.synchronize(); print(p[:4].tolist())
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fc_tc -c 1 -o gpurun_out/r2d/fctc python /tmp/one.py > gpurun_out/r2d/ncu.log 2>&1
tail -3 gpurun_out/r2d/ncu.log

# functional check of bench.py's multi-rank path on one GPU (gloo; two ranks share cuda:0): not a measurement
O=gpurun_out/r2z; mkdir -p $O
TNB_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 > $O/b2.log 2>&1; echo "2-rank exit $?"; tail -1 $O/b2.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref.log 2>&1; echo "ref exit $?"; tail -1 $O/ref.log | cut -c1-300

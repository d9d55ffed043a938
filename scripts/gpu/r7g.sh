# strong-scaling estimate on one GPU: rank 0's block of a G-GPU run timed alone (G = 1, 2, 4, 8)
O=gpurun_out/r7g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for wl in C5a C4b; do timeout 600 python scripts/scaling_estimate.py $wl > $O/scaling_$wl.json 2> $O/scaling_$wl.err; cat $O/scaling_$wl.json; done

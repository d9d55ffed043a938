set -x; O=gpurun_out/${TAG:-r1m}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python scripts/plan_bench.py --workload C5a --recipes "4,rgreedy-fill,8,0.3,0;5,rgreedy-fill,8,0.3,0;5,rgreedy-fill,16,0.2,5;7,rgreedy-fill,16,0.2,5;4,rgreedy-fill,16,0.3,2;3,rgreedy-fill,16,0.3,3;6,rgreedy-fill,8,0.3,0" > $O/plans.log 2>&1; echo "plans exit $?"; cat $O/plans.log

# C5a plan recipes with CUDA graphs: the r = n pick vs the r = 4 multi-round candidates
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python scripts/recipe_bench.py --orderer rgreedy-fill --k 5 --q 16 --tau 0.2 --seed 5
timeout 300 python scripts/recipe_bench.py --orderer rgreedy-fill --k 6 --q 16 --tau 0.3 --seed 2 --r 4
timeout 300 python scripts/recipe_bench.py --orderer rgreedy-fill --k 8 --q 16 --tau 0.3 --seed 2 --r 4
timeout 300 python scripts/recipe_bench.py --orderer rgreedy-fill --k 5 --q 16 --tau 0.3 --seed 4 --r 4
TNB_GRAPH=0 timeout 300 python scripts/recipe_bench.py --orderer rgreedy-fill --k 6 --q 16 --tau 0.3 --seed 2 --r 4

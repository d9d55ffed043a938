# k_gemm_fc: 4 x 2 register blocks with the consumer loads at the start of the tile vs the 4 x 4 default
python -c "import __graft_entry__ as g; g.build()"
for v in 2 1; do for wb in 3 2; do
TNB_FC_RBB=$v TNB_FC_WB=$wb timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2y_$v$wb.json 2> gpurun_out/r2y_$v$wb.err
python -c "
import json; d=json.load(open('gpurun_out/r2y_$v$wb.json')); r=d['roofline']; print('RBB=$v WB=$wb', d['value'], json.dumps({k:(round(x['ms_share_of_step'],3), round(x['GBps'])) for k,x in r['families'].items()}))"
done; done

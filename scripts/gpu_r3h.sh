O=gpurun_out/r3h; mkdir -p $O
for I in 0 1 3; do TNB_RECIPE_INDEX=$I timeout 900 python tests/run_configs.py --only C4b --out $O/c4b_$I.json > $O/c4b_$I.log 2>&1; python -c "import json;d=json.loads(open('$O/c4b_$I.log').read().strip().splitlines()[-1]);print('recipe $I', d['k'], d['width'], d['ms_per_contraction_c64'], d.get('slice_parity'), d.get('closed_form_rel_err_c64'))"; done

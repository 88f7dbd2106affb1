# round 2, call bj: grouped plan (identity components joined into one copy-through component)
# -- full GPU suite, same-box A/B against ADHA_GROUP_IDENTITY=0 on the bench configs
set -u
out=gpurun_out
timeout 2000 python -m pytest tests -m gpu -q -x > $out/bj_pytest.log 2>&1; echo "pytest=$?"
for round in 1 2; do
  for g in 0 1; do
    for c in C3 C3R P1 C4 P2; do
      ADHA_GROUP_IDENTITY=$g python bench.py --config $c --no-cpu-baseline --no-e2e --sustained-s 0 > $out/bj_g${g}_${c}_$round.json 2>/dev/null
      python -c "import json;d=json.load(open('$out/bj_g${g}_${c}_$round.json'));print('group=$g $c round $round', round(d['value'],1), round(d['frac_of_same_run_copy'],4))" >> $out/bj_ab.log
    done
  done
done
timeout 900 python tools/merge_probe.py > $out/bj_merge_probe.log 2>&1; echo "probe=$?"

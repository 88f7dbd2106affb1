# round 2, call br: store evict_first hints (ADHA_L2_HINTS=2) on the bench lines (whole chains)
set -u
out=gpurun_out
for round in 1 2; do
  for h in 0 2; do
    for c in C4 P1 C4M C5 C2; do
      ADHA_L2_HINTS=$h python bench.py --config $c --no-cpu-baseline --no-e2e --sustained-s 0 > $out/br_h${h}_${c}_$round.json 2>/dev/null
      python -c "import json;d=json.load(open('$out/br_h${h}_${c}_$round.json'));print('hints=$h $c round $round', round(d['value'],1), round(d['frac_of_same_run_copy'],4))" >> $out/br_ab.log
    done
  done
done

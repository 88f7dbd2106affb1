# round 2, call am: TMA write-back (ADHA_COPYOUT=tma) vs consumer STG on the chain / moved-subset
# configs whose dst chunks per tile are few (C4M: 3 x 16 KB; P1 hop 0: 2)
set -u
out=gpurun_out
for round in 1 2; do
  for m in auto tma; do
    for c in C4M P1 C4 P2; do
      ADHA_COPYOUT=$m python bench.py --config $c --no-cpu-baseline --no-e2e --sustained-s 0 > $out/am_${m}_${c}_$round.json 2>/dev/null
      python -c "import json;d=json.load(open('$out/am_${m}_${c}_$round.json'));print('copyout=$m $c round $round', round(d['value'],1), round(d['frac_of_same_run_copy'],4))" >> $out/am_ab.log
    done
  done
done

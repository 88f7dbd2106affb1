# round 2, call bg: merged plan without a size limit for <= 8 src clusters (Medical AoSV -> SoA in
# C4 and P1): bench A/B against the former 64 MB limit (ADHA_MERGE_BYTES=67108864)
set -u
out=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "chain or regions or full_size" > $out/bg_pytest.log 2>&1; echo "pytest=$?"
for round in 1 2; do
  for v in old new; do
    for c in P1 C4 P2; do
      if [ $v = old ]; then export ADHA_MERGE_BYTES=67108864; else unset ADHA_MERGE_BYTES; fi
      python bench.py --config $c --no-cpu-baseline --no-e2e --sustained-s 0 > $out/bg_${v}_${c}_$round.json 2>/dev/null
      python -c "import json;d=json.load(open('$out/bg_${v}_${c}_$round.json'));print('$v $c round $round', round(d['value'],1), round(d['frac_of_same_run_copy'],4))" >> $out/bg_ab.log
    done
  done
done
unset ADHA_MERGE_BYTES
CFGS=C4,P1 ROUNDS=5 timeout 900 python tools/ab_multi.py "ADHA_MERGE_BYTES=67108864" "" > $out/bg_edges.log 2>&1; echo "ab=$?"

# round 2, call bd: PDL trigger at the second-to-last tile (trig2) vs the last tile (cur)
# tile) vs without (dependents scheduled as CTAs exit); same box, alternating libraries
set -u
out=gpurun_out
cp paper_1407_4859_b200/libadha.so /tmp/libadha_cur.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "chain or pairs or capture" > $out/bd_pytest.log 2>&1; echo "pytest=$?"
for round in 1 2; do
  for v in trig2 cur; do
    if [ $v = cur ]; then cp /tmp/libadha_cur.so paper_1407_4859_b200/libadha.so; else cp paper_1407_4859_b200/_build/trig2/libadha.so paper_1407_4859_b200/libadha.so; fi
    for c in C2 P1 C4M P2 C4; do
      python bench.py --config $c --no-cpu-baseline --no-e2e --sustained-s 0 > $out/bd_${v}_${c}_$round.json 2>/dev/null
      python -c "import json;d=json.load(open('$out/bd_${v}_${c}_$round.json'));print('$v $c round $round', round(d['value'],1), round(d['frac_of_same_run_copy'],4))" >> $out/bd_ab.log
    done
  done
done
cp /tmp/libadha_cur.so paper_1407_4859_b200/libadha.so

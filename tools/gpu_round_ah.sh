# round 2, call ah: same-box A/B of the round's start library (48073bc, _build/old) against the
# current one on the bench configs (burst value), and the small-path sweep of the current build
set -u
out=gpurun_out
cp paper_1407_4859_b200/libadha.so /tmp/libadha_cur.so
for round in 1 2; do
  for v in old cur; do
    if [ $v = cur ]; then cp /tmp/libadha_cur.so paper_1407_4859_b200/libadha.so; else cp paper_1407_4859_b200/_build/old/libadha.so paper_1407_4859_b200/libadha.so; fi
    for c in C5 C4M C2 P1; do
      python bench.py --config $c --no-cpu-baseline --no-e2e --sustained-s 0 > $out/ah_${v}_${c}_$round.json 2>/dev/null
      python -c "import json;d=json.load(open('$out/ah_${v}_${c}_$round.json'));print('$v $c round $round', round(d['value'],1), round(d['frac_of_same_run_copy'],4))" >> $out/ah_ab.log
    done
  done
done
cp /tmp/libadha_cur.so paper_1407_4859_b200/libadha.so
timeout 900 python tools/small_path_probe.py "C3 SoA->hybrid (64 f)" "K-Means SoA->AoS (32 f)" "C2 AoS->SoA" > $out/ah_small_path.log 2>&1; echo "small=$?"

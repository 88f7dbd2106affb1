# round 2, call av: programmatic dependent launch of the tiled kernel (ADHA_PDL) -- tests, A/B
set -u
out=gpurun_out
timeout 2000 python -m pytest tests -m gpu -q -x > $out/av_pytest.log 2>&1; echo "pytest=$?"
for round in 1 2; do
  for pdl in 0 1; do
    for c in C2 P1 C4 C4M P2 C5; do
      ADHA_PDL=$pdl python bench.py --config $c --no-cpu-baseline --no-e2e --sustained-s 0 > $out/av_p${pdl}_${c}_$round.json 2>/dev/null
      python -c "import json;d=json.load(open('$out/av_p${pdl}_${c}_$round.json'));print('pdl=$pdl $c round $round', round(d['value'],1), round(d['frac_of_same_run_copy'],4))" >> $out/av_ab.log
    done
  done
done
for pdl in 0 1; do ADHA_PDL=$pdl timeout 900 python tools/small_path_probe.py "C2 AoS->SoA" "C3 SoA->hybrid (64 f)" "Medical AoSV->SoA" > $out/av_small_p$pdl.log 2>&1; done; echo "small=$?"

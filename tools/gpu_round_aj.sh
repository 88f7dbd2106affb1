# round 2, call aj: unit-mode permutation items balanced over the consumer warps (ADHA_UNIT_BALANCE)
set -u
out=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_inplace.py -m gpu -q -x -k "not max_size" > $out/aj_pytest.log 2>&1; echo "pytest=$?"
for round in 1 2; do
  for b in 0 1; do
    for c in C5 C4M C2 P1 C4; do
      ADHA_UNIT_BALANCE=$b python bench.py --config $c --no-cpu-baseline --no-e2e --sustained-s 2 > $out/aj_b${b}_${c}_$round.json 2>/dev/null
      python -c "import json;d=json.load(open('$out/aj_b${b}_${c}_$round.json'));print('balance=$b $c round $round', round(d['value'],1), round(d['frac_of_same_run_copy'],4), 'sustained', round(d['sustained']['value'],1), d['sustained']['clocks']['sm_mhz'])" >> $out/aj_ab.log
    done
  done
done
for b in 0 1; do echo "== ADHA_UNIT_BALANCE=$b" >> $out/aj_phase.log; ADHA_UNIT_BALANCE=$b python tools/phase_probe.py >> $out/aj_phase.log 2>&1; done; echo "phase=$?"

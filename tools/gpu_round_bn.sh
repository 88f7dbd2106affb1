# round 2, call bn: programmatic dependent launch for the in-place kernels -- tests, stress, A/B
set -u
out=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_inplace.py tests/test_gpu_bench.py -m gpu -q -x > $out/bn_pytest.log 2>&1; echo "pytest=$?"
ADHA_IP_VERIFY=1 timeout 1200 python tools/stress_inplace.py 500 5028 > $out/bn_stress_inplace.log 2>&1; echo "stress=$?"
for round in 1 2; do
  for pdl in 0 1; do
    for c in C2 C4 P2; do
      ADHA_PDL=$pdl python bench.py --inplace --config $c --no-cpu-baseline --no-e2e > $out/bn_p${pdl}_${c}_$round.json 2>/dev/null
      python -c "import json;d=json.load(open('$out/bn_p${pdl}_${c}_$round.json'));print('pdl=$pdl $c round $round', round(d['value'],1))" >> $out/bn_ab.log
    done
  done
done

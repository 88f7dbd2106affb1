# round 2, call bm: programmatic dependent launch for the direct kernel and the fused small chain
set -u
out=gpurun_out
timeout 2000 python -m pytest tests -m gpu -q -x > $out/bm_pytest.log 2>&1; echo "pytest=$?"
for pdl in 0 1; do ADHA_PDL=$pdl timeout 900 python tools/small_path_probe.py "C2 AoS->SoA" "Medical AoSV->SoA" "C3 SoA->hybrid (64 f)" > $out/bm_small_p$pdl.log 2>&1; done; echo "small=$?"
for pdl in 0 1; do for r in 1 2; do ADHA_PDL=$pdl python bench.py --config C1 --no-cpu-baseline --no-e2e --sustained-s 0 > $out/bm_c1_p${pdl}_$r.json 2>/dev/null; done; done; echo "c1=$?"

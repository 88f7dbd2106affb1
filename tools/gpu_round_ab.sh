# round 2, call ab: consumer cp.async loader (ADHA_LOADER=cpa) -- parity with it forced on, A/B
# against the TMA producer over the bench edges, and the small/mid-size sweep with it
set -u
out=gpurun_out
ADHA_LOADER=cpa timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $out/ab_pytest_cpa.log 2>&1; echo "pytest=$?"
CFGS=C5,C2,C3,C3R,C4,P1,P2 ROUNDS=5 timeout 900 python tools/ab_multi.py "" "ADHA_LOADER=cpa" > $out/ab_loader.log 2>&1; echo "ab=$?"
ADHA_LOADER=cpa timeout 900 python tools/small_path_probe.py > $out/ab_small_path_cpa.log 2>&1; echo "small=$?"

# round 2, call at: cp.async loader as NLOAD=3 dedicated loader warps (TMA producer's protocol)
set -u
out=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "loaders or capture" > $out/at_pytest.log 2>&1; echo "pytest=$?"
ADHA_LOADER=cpa timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "not full_size and not max_size and not large_n" > $out/at_pytest_cpa.log 2>&1; echo "pytest cpa=$?"
CFGS=C5,C2,C3,C4,P1,P2 ROUNDS=5 timeout 900 python tools/ab_multi.py "" "ADHA_LOADER=cpa" > $out/at_loader.log 2>&1; echo "ab=$?"
ADHA_LOADER=cpa timeout 900 python tools/small_path_probe.py "C2 AoS->SoA" "K-Means SoA->AoS (32 f)" "C3 SoA->hybrid (64 f)" "C3 hybrid->SoA (64 f)" "Medical AoSV->SoA" > $out/at_small_path_cpa.log 2>&1; echo "small=$?"

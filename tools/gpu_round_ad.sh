# round 2, call ad: loader tests (tma / cpa forced, merged and component plans), auto rule sweep
set -u
out=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "loaders or capture or write_back" > $out/ad_pytest.log 2>&1; echo "pytest=$?"
timeout 900 python tools/small_path_probe.py "K-Means SoA->AoS (32 f)" "C3 SoA->hybrid (64 f)" "C2 AoS->SoA" > $out/ad_small_path.log 2>&1; echo "small=$?"

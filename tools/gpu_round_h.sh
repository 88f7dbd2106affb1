# round 2, call h: remap_host mirror mode (parity + e2e sweeps)
set -u
out=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "remap_host" > $out/h_pytest.log 2>&1; echo "pytest=$?"
MODES="mirror zero hybrid" CBS="67108864 268435456" bash tools/e2e_sweep.sh C3 > $out/h_e2e_c3.log 2>&1; echo "c3=$?"
MODES="mirror zero hybrid" CBS="67108864 268435456" bash tools/e2e_sweep.sh C3R > $out/h_e2e_c3r.log 2>&1; echo "c3r=$?"
MODES="mirror hybrid" CBS="16777216 67108864" bash tools/e2e_sweep.sh C2 > $out/h_e2e_c2.log 2>&1; echo "c2=$?"
MODES="mirror hybrid" CBS="16777216 67108864" bash tools/e2e_sweep.sh P2 > $out/h_e2e_p2.log 2>&1; echo "p2=$?"

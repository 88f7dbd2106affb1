# round 2, call s: byte-group slots balanced over the warps (I = 3, 5, 6, 7 with GMAX 2)
set -u
out=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > $out/s_pytest.log 2>&1; echo "pytest=$?"
python tools/narrow_probe.py > $out/s_narrow_probe.log 2>&1; echo "narrow=$?"
python tools/phase_probe.py > $out/s_phase.log 2>&1; echo "phase=$?"
timeout 600 python tools/small_path_probe.py "g2 [2,4,6,4]x4 AoS->SoA" "narrow 24x1B+8 AoS->SoA" > $out/s_small.log 2>&1; echo "small=$?"

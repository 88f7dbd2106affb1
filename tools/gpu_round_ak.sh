# round 2, call ak: byte-group (instruction, period) items split over the warps by the planner's
# per-instruction cost instead of by count; narrow-field parity, probe, phase probe
set -u
out=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "byte or pairs or generalised or narrow or config_shapes or write_back" > $out/ak_pytest.log 2>&1; echo "pytest=$?"
for i in 1 2; do python tools/narrow_probe.py >> $out/ak_narrow_probe.log 2>&1; done; echo "narrow=$?"
python tools/phase_probe.py > $out/ak_phase.log 2>&1; echo "phase=$?"
timeout 600 python tools/small_path_probe.py "g2 [2,4,6,4]x4 AoS->SoA" "narrow 24x1B+8 AoS->SoA" > $out/ak_small.log 2>&1; echo "small=$?"

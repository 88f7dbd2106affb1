# round 2, call as: phase breakdown of the small/mid-size tiled launches with the final library
set -u
out=gpurun_out
python tools/phase_probe.py --small > $out/as_phase_small.log 2>&1; echo "phase=$?"
ADHA_LOADER=tma python tools/phase_probe.py --small > $out/as_phase_small_tma.log 2>&1; echo "phase tma=$?"
ADHA_LOADER=cpa python tools/phase_probe.py --small > $out/as_phase_small_cpa.log 2>&1; echo "phase cpa=$?"

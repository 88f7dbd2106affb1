# round 2, call bp: C3 SoA->hybrid mid-size -- smaller merged tiles / more stages, both loaders
set -u
out=gpurun_out
for sb in 49152 24576 16384; do
  for ld in tma cpa; do
    echo "== stage $sb loader $ld" >> $out/bp_c3_mid.log
    ADHA_STAGE_BYTES=$sb ADHA_STAGES=6 ADHA_LOADER=$ld timeout 600 python tools/small_path_probe.py "C3 SoA->hybrid (64 f)" 2>&1 | grep -E '"payload_MB": (8.0|16.0|32.0|128.0)' >> $out/bp_c3_mid.log
  done
done

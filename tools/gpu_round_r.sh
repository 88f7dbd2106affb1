# round 2, call r: merged-plan stage size for many-region shapes (C3 at 32-128 MB)
set -u
out=gpurun_out
for v in "base:" "st64k:ADHA_STAGE_BYTES=65536" "st64k_o1:ADHA_STAGE_BYTES=65536 ADHA_OUT_BUFFERS=1" "st96k_o1:ADHA_STAGE_BYTES=98304 ADHA_OUT_BUFFERS=1" "st32k:ADHA_STAGE_BYTES=32768" "stages3_32k:ADHA_STAGE_BYTES=32768 ADHA_STAGES=3"; do
  tag=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python tools/small_path_probe.py "C3 SoA->hybrid (64 f)" "C3 hybrid->SoA (64 f)" "C2 AoS->SoA" > $out/r_small_$tag.log 2>&1; echo "$tag=$?"
done

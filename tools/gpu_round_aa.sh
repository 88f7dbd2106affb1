# round 2, call aa: many-region tiles -- TMA bulk copies per piece vs consumer cp.async (LDGSTS),
# at 32 MiB (mid-size) and 2 GiB (tools/copy_probe.cu "pieces")
set -u
out=gpurun_out
for g in 0.03125 2; do
  echo "== $g GiB" >> $out/aa_pieces.log
  timeout 300 tools/copy_probe $g pieces >> $out/aa_pieces.log 2>&1; echo "probe $g=$?"
done

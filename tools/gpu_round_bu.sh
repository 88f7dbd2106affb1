# round 2, call bu: zero-copy e2e (kernel reads pinned host memory) vs stage size / count
set -u
out=gpurun_out
for spec in "49152 2" "24576 6" "16384 8" "32768 4"; do
  set -- $spec
  for c in C3 C2; do
    r=$(ADHA_STAGE_BYTES=$1 ADHA_STAGES=$2 ADHA_HOST_MODE=zero timeout 300 python bench.py --config $c --no-cpu-baseline --no-copy-ref --sustained-s 0 --steps 10 2>/dev/null | tail -1)
    python -c "import json,sys; d=json.loads(sys.argv[1]); print('stage $1 x $2 $c zero e2e %.1f GB/s' % d['e2e']['value'])" "$r" >> $out/bu_e2e.log || echo "$1 $2 $c ERR" >> $out/bu_e2e.log
  done
done

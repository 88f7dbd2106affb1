#!/bin/bash
# e2e (host buffers through adha_remap_host) per mode and chunk size
cfg=${1:-C2}
for mode in ${MODES:-zero hybrid staged}; do
  for cb in ${CBS:-16777216 33554432 67108864}; do
    out=$(ADHA_HOST_MODE=$mode ADHA_HOST_CHUNK_BYTES=$cb timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-copy-ref --sustained-s 0 --steps 10 2>&1 | tail -1)
    python -c "import json,sys; d=json.loads(sys.argv[3]); print(sys.argv[1], sys.argv[2], 'e2e %.1f GB/s' % d['e2e']['value'], '%.2f ms/step' % d['e2e']['ms_per_step'])" $mode $cb "$out" || echo "$mode $cb ERR"
    [ $mode = zero ] && break
  done
done

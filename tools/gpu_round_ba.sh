# round 2, call ba: zero-copy e2e (kernel reads pinned host src) with the cp.async loader warps
# instead of TMA bulk copies over PCIe
set -u
out=gpurun_out
for ld in tma cpa; do
  for c in C3 C2; do
    for mode in zero; do
      r=$(ADHA_LOADER=$ld ADHA_HOST_MODE=$mode timeout 300 python bench.py --config $c --no-cpu-baseline --no-copy-ref --sustained-s 0 --steps 5 2>/dev/null | tail -1)
      python -c "import json,sys; d=json.loads(sys.argv[1]); print('$ld $c $mode e2e %.1f GB/s' % d['e2e']['value'])" "$r" >> $out/ba_e2e.log || echo "$ld $c $mode ERR" >> $out/ba_e2e.log
    done
  done
done

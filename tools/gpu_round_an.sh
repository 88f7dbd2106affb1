# round 2, call an: remap_host with all H2D copies in chunk order on one stream (kernels per slot)
set -u
out=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "remap_host or host_threads" > $out/an_pytest.log 2>&1; echo "pytest=$?"
for c in C5 C2 C3; do
  echo "== $c" >> $out/an_e2e.log
  MODES="hybrid" CBS="16777216 67108864 268435456" bash tools/e2e_sweep.sh $c >> $out/an_e2e.log 2>&1
  MODES="zero" bash tools/e2e_sweep.sh $c >> $out/an_e2e.log 2>&1
  python bench.py --config $c --no-cpu-baseline --no-copy-ref --sustained-s 0 --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default e2e %.1f GB/s' % d['e2e']['value'])" >> $out/an_e2e.log
done

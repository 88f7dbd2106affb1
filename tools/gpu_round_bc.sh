# round 2, call bc: e2e vs --steps (zero-copy C2, hybrid C5)
set -u
out=gpurun_out
for spec in "C2 zero" "C2 auto" "C5 auto"; do
  set -- $spec
  for k in 3 5 10; do
    r=$(ADHA_HOST_MODE=$2 timeout 300 python bench.py --config $1 --no-cpu-baseline --no-copy-ref --sustained-s 0 --steps $k --warmup 3 2>/dev/null | tail -1)
    python -c "import json,sys; d=json.loads(sys.argv[1]); print('$1 $2 steps $k e2e %.1f GB/s' % d['e2e']['value'], d['e2e'].get('ms_per_step'))" "$r" >> $out/bc_e2e.log || echo "$1 $2 $k ERR" >> $out/bc_e2e.log
  done
done

# round 2, call bb: e2e A/B of the round's starting library vs the current one (same box): auto mode
# (C3: zero-copy, C2: hybrid) and zero mode for C2
set -u
out=gpurun_out
cp paper_1407_4859_b200/libadha.so /tmp/libadha_cur.so
for round in 1 2; do
  for v in old cur; do
    if [ $v = cur ]; then cp /tmp/libadha_cur.so paper_1407_4859_b200/libadha.so; else cp paper_1407_4859_b200/_build/old/libadha.so paper_1407_4859_b200/libadha.so; fi
    for spec in "C3 auto" "C2 auto" "C2 zero"; do
      set -- $spec
      r=$(ADHA_HOST_MODE=$2 timeout 300 python bench.py --config $1 --no-cpu-baseline --no-copy-ref --sustained-s 0 --steps 10 2>/dev/null | tail -1)
      python -c "import json,sys; d=json.loads(sys.argv[1]); print('$v $1 $2 round $round e2e %.1f GB/s' % d['e2e']['value'])" "$r" >> $out/bb_e2e.log || echo "$v $1 $2 ERR" >> $out/bb_e2e.log
    done
  done
done
cp /tmp/libadha_cur.so paper_1407_4859_b200/libadha.so

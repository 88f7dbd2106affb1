for st in 50 400 50 400; do
  for soak in 1.5 0; do
    python bench.py --steps $st --soak-s $soak --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('steps $st soak $soak', round(d['value']), 'copy', round(d['same_run_copy_gbs_per_gpu']), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'spread', round(d['step_ms_spread']['median'],4))"
  done
done

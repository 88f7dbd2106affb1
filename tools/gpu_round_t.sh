# round 2, call t: experiment -- pipelined STG write-back (ADHA_PIPE=1) vs sequential (0); the
# library spills registers in this build, so both legs run the same (spilling) binary
set -u
out=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config_shapes or all_layout_pairs or full_size_exact" > $out/t_pytest.log 2>&1; echo "pytest=$?"
for pp in 1 0; do
  for c in C5 C2 P1 C4M; do
    ADHA_PIPE=$pp python bench.py --config $c --no-cpu-baseline --no-e2e --sustained-s 3 > $out/t_bench_${c}_pipe$pp.json 2> $out/t_bench_${c}_pipe$pp.err; echo "bench $c pipe$pp=$?"
  done
  ADHA_PIPE=$pp python tools/phase_probe.py > $out/t_phase_pipe$pp.log 2>&1; echo "phase pipe$pp=$?"
done

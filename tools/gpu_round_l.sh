# round 2, call l: fused chain with deferred store fences and division-free tile iteration
set -u
out=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "chain" > $out/l_pytest_chain.log 2>&1; echo "pytest chain=$?"
for c in C4 P1 P2; do
  for g in 4 8; do
    ADHA_CHAIN_GROUP=$g python bench.py --config $c --no-cpu-baseline --sustained-s 0 --no-e2e --no-copy-ref > $out/l_bench_${c}_g$g.json 2> $out/l_bench_${c}_g$g.err; echo "bench $c g$g=$?"
  done
  ADHA_CHAIN_TILED_BYTES=0 python bench.py --config $c --no-cpu-baseline --sustained-s 0 --no-e2e --no-copy-ref > $out/l_bench_${c}_unfused.json 2> $out/l_bench_${c}_unfused.err; echo "bench $c unfused=$?"
done
python bench.py --config C4 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-copy-ref --sustained-s 0 > $out/l_plain.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:remap_tiled -s 3 -c 1 -o $out/l_prof_c4chain \
      python bench.py --config C4 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-copy-ref --sustained-s 0 > /dev/null 2>&1
echo "ncu=$?"

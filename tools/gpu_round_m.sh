# round 2, call m: fused chain L2 hints; burst and power-capped (sustained) regimes
set -u
out=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "chain" > $out/m_pytest_chain.log 2>&1; echo "pytest chain=$?"
for c in C4 P2; do
  for v in "g4h1:ADHA_CHAIN_GROUP=4 ADHA_CHAIN_HINTS=1" "g8h1:ADHA_CHAIN_GROUP=8 ADHA_CHAIN_HINTS=1" "g8h0:ADHA_CHAIN_GROUP=8 ADHA_CHAIN_HINTS=0" "g6h1:ADHA_CHAIN_GROUP=6 ADHA_CHAIN_HINTS=1" "unfused:ADHA_CHAIN_TILED_BYTES=0"; do
    tag=${v%%:*}; envs=${v#*:}
    env $envs python bench.py --config $c --no-cpu-baseline --no-e2e --sustained-s 3 > $out/m_bench_${c}_$tag.json 2> $out/m_bench_${c}_$tag.err; echo "bench $c $tag=$?"
  done
done
ADHA_CHAIN_GROUP=8 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none \
   -k regex:remap_tiled -s 4 -c 2 --csv --log-file $out/m_steady_C4_g8.csv \
   python bench.py --config C4 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-copy-ref --sustained-s 0 > /dev/null 2>&1
echo "ncu=$?"

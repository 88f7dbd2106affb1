# round 2, call j: fused tiled chain (one launch, intermediates read back from L2)
set -u
out=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "chain" > $out/j_pytest_chain.log 2>&1; echo "pytest chain=$?"
for c in C4 P1 P2; do
  python bench.py --config $c --no-cpu-baseline --sustained-s 0 --no-e2e > $out/j_bench_$c.json 2> $out/j_bench_$c.err; echo "bench $c=$?"
  ADHA_CHAIN_TILED_BYTES=0 python bench.py --config $c --no-cpu-baseline --sustained-s 0 --no-e2e > $out/j_bench_${c}_unfused.json 2> $out/j_bench_${c}_unfused.err; echo "bench $c unfused=$?"
done
python bench.py --config C4 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-copy-ref --sustained-s 0 > $out/j_plain.log 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum --cache-control none --clock-control none \
      -k regex:remap_tiled -s 4 -c 2 --csv --log-file $out/j_steady_C4.csv \
      python bench.py --config C4 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-copy-ref --sustained-s 0 > /dev/null 2>&1
echo "ncu=$?"
timeout 900 python -m pytest tests -m gpu -q -x > $out/j_pytest.log 2>&1; echo "pytest=$?"

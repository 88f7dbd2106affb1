# round 2, call o: chain mode as its own template instantiation (plain kernels without chain code)
set -u
out=gpurun_out
timeout 2000 python -m pytest tests -m gpu -q -x > $out/o_pytest.log 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $out/o_smoke.log 2>&1; echo "smoke=$?"
for c in C5 C2 C3 C4 C4M P1; do
  python bench.py --config $c --no-cpu-baseline --sustained-s 0 --no-e2e > $out/o_bench_$c.json 2> $out/o_bench_$c.err; echo "bench $c=$?"
done
for c in C2 C4M; do
  ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,smsp__inst_executed.sum --cache-control none --clock-control none \
     -k regex:remap_tiled -s 4 -c 2 --csv --log-file $out/o_steady_$c.csv \
     python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-copy-ref --sustained-s 0 > /dev/null 2>&1
  echo "ncu $c=$?"
done
ADHA_CHAIN_TILED_BYTES=67108864 python bench.py --config C4 --no-cpu-baseline --sustained-s 0 --no-e2e > $out/o_bench_C4_fused.json 2> $out/o_bench_C4_fused.err; echo "bench C4 fused=$?"

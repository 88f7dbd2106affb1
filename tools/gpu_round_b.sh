# round 2, call b: parity after the shared-memory entry table, small/mid-size A/B, benches,
# steady-state DRAM traffic (cache-control none, a launch in the middle of back-to-back launches)
set -u
out=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > $out/b_pytest.log 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $out/b_smoke.log 2>&1; echo "smoke=$?"
timeout 600 python tools/small_path_probe.py > $out/b_small_path.log 2>&1; echo "small=$?"
for c in C5 C2 C3 C3R C4 P1 P2; do
  python bench.py --config $c --no-cpu-baseline --sustained-s 0 > $out/b_bench_$c.json 2> $out/b_bench_$c.err; echo "bench $c=$?"
done
for c in C2 P1 C5; do
  python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-copy-ref --sustained-s 0 > $out/b_plain_$c.log 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none \
      -k regex:remap_tiled -s 4 -c 3 --csv --log-file $out/b_steady_$c.csv \
      python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-copy-ref --sustained-s 0 > /dev/null 2>&1
  echo "steady $c=$?"
done

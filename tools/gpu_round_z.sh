# round 2, call z: plan tables in device memory (coalesced copy to shared memory, ~7 KB kernel
# parameters instead of up to 31 KB): GPU tests, small-path sweep, default bench lines
set -u
out=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > $out/z_pytest.log 2>&1; echo "pytest=$?"
timeout 900 python tools/small_path_probe.py > $out/z_small_path.log 2>&1; echo "small=$?"
for c in C5 C2 C3 C4M; do
  python bench.py --config $c --no-cpu-baseline --no-e2e > $out/z_bench_$c.json 2> $out/z_bench_$c.err; echo "bench $c=$?"
done

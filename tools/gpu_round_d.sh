# round 2, call d: merged one-component plan for small / mid-size multi-component remaps
set -u
out=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > $out/d_pytest.log 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $out/d_smoke.log 2>&1; echo "smoke=$?"
timeout 900 python tools/small_path_probe.py > $out/d_small_path.log 2>&1; echo "small=$?"
python tools/phase_probe.py --small > $out/d_phase_small.log 2>&1; echo "phase=$?"
for c in C3 C4M; do
  python bench.py --config $c --no-cpu-baseline --sustained-s 0 > $out/d_bench_$c.json 2> $out/d_bench_$c.err; echo "bench $c=$?"
done

# round 2, call i: one-component plans read their entries from the parameters again
set -u
out=gpurun_out
timeout 2000 python -m pytest tests -m gpu -q -x > $out/i_pytest.log 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $out/i_smoke.log 2>&1; echo "smoke=$?"
timeout 900 python tools/small_path_probe.py "C2 AoS->SoA" "C2 SoA->AoS" "Medical AoS->AoSV" "K-Means 4xAoS8->AoS" "C3 SoA->hybrid (64 f)" > $out/i_small_path.log 2>&1; echo "small=$?"
for c in C5 C2 P1; do
  python bench.py --config $c --no-cpu-baseline --sustained-s 0 --no-e2e > $out/i_bench_$c.json 2> $out/i_bench_$c.err; echo "bench $c=$?"
done

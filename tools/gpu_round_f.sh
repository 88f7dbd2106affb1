# round 2, call f: LDGSTS producer for small src chunks, tail spreading
set -u
out=gpurun_out
timeout 2000 python -m pytest tests -m gpu -q -x > $out/f_pytest.log 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $out/f_smoke.log 2>&1; echo "smoke=$?"
timeout 900 python tools/small_path_probe.py > $out/f_small_path.log 2>&1; echo "small=$?"
python tools/phase_probe.py --small > $out/f_phase_small.log 2>&1; echo "phase=$?"
timeout 900 env ADHA_IP_VERIFY=1 python tools/stress_inplace.py 300 > $out/f_stress_inplace.log 2>&1; echo "stress=$?"
for c in C3 C3R C5; do
  python bench.py --config $c --no-cpu-baseline --sustained-s 0 > $out/f_bench_$c.json 2> $out/f_bench_$c.err; echo "bench $c=$?"
done
CBS="67108864 268435456" bash tools/e2e_sweep.sh C3 > $out/f_e2e_c3.log 2>&1; echo "e2e sweep=$?"

# round 2, call e: 128-bit table copy, merged plan, faster in-place host plan
set -u
out=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > $out/e_pytest.log 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $out/e_smoke.log 2>&1; echo "smoke=$?"
timeout 600 ADHA_IP_VERIFY=1 python tools/stress_inplace.py 300 > $out/e_stress_inplace.log 2>&1; echo "stress=$?"
timeout 900 python tools/small_path_probe.py > $out/e_small_path.log 2>&1; echo "small=$?"
python tools/phase_probe.py --small > $out/e_phase_small.log 2>&1; echo "phase=$?"
python tools/one_remap.py c3 1 > $out/e_one_c3.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:remap_tiled -s 2 -c 1 -o $out/e_prof_c3 \
      python tools/one_remap.py c3 1 > $out/e_ncu_c3.log 2>&1
echo "ncu=$?"
for c in C2 C3; do
  python bench.py --inplace --config $c > $out/e_bench_inplace_$c.json 2> $out/e_bench_inplace_$c.err; echo "inplace $c=$?"
done
python bench.py > $out/e_bench_C5.json 2> $out/e_bench_C5.err; echo "bench=$?"

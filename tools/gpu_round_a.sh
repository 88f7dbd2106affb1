set -u
out=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/g1_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $out/g1_smoke.log 2>&1; echo "smoke=$?"
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > $out/g1_pytest.log 2>&1; echo "pytest=$?"
python bench.py > $out/g1_bench.json 2> $out/g1_bench.err; echo "bench=$?"
python bench.py --config C4M --no-cpu-baseline > $out/g1_bench_C4M.json 2> $out/g1_bench_C4M.err; echo "c4m=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --sustained-s 0 > $out/g1_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/g1_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --sustained-s 0 > $out/g1_ncu_launch.log 2>&1
echo "ncu=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $out/g1_smoke2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --csv --log-file $out/g1_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
echo "smoke ncu=$?"

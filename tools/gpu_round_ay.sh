# round 2, call ay: the final tree (after PDL and the re-placed thresholds) -- full GPU suite, smoke and its launch list, default bench line
set -u
out=gpurun_out
tag=r02ay
timeout 2000 python -m pytest tests -m gpu -q > $out/${tag}_pytest.log 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --csv --log-file $out/${tag}_smoke_launches.csv \
      python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
echo "smoke=$?"
python bench.py > $out/bench_${tag}.json 2> $out/bench_${tag}.err; echo "bench=$?"
python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_${tag}_reference.json 2>&1; echo "reference=$?"
timeout 600 python tools/small_path_probe.py "C2 AoS->SoA" "K-Means SoA->AoS (32 f)" "C3 SoA->hybrid (64 f)" "Medical AoSV->SoA" > $out/${tag}_small_path.log 2>&1; echo "small=$?"

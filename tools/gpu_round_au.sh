# round 2, call au: the final tree -- full GPU suite, smoke and its launch list, default bench line
set -u
out=gpurun_out
tag=r02au
timeout 2000 python -m pytest tests -m gpu -q > $out/${tag}_pytest.log 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --csv --log-file $out/${tag}_smoke_launches.csv \
      python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
echo "smoke=$?"
python bench.py > $out/bench_${tag}.json 2> $out/bench_${tag}.err; echo "bench=$?"
python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_${tag}_reference.json 2>&1; echo "reference=$?"

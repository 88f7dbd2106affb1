# round 2, call bo (final tree: PDL on every remap kernel; bi, ax, al, ag, g before it): GPU evidence of the round's state -- parity, smoke (+ its launch list),
# every bench line, the launch list of the default bench, ncu --set full of the remap kernel
# per config, steady-state traffic, small/mid-size sweep, tuning profile, in-place lines
set -u
tag=${1:-r02bo}
out=gpurun_out
timeout 2000 python -m pytest tests -m gpu -q > $out/${tag}_pytest.log 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --csv --log-file $out/${tag}_smoke_launches.csv \
      python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
echo "smoke=$?"
python bench.py > $out/bench_${tag}.json 2> $out/bench_${tag}.err; echo "bench=$?"
for c in C1 C2 C3 C3R C4 C4M P1 P2; do
  python bench.py --config $c --no-cpu-baseline > $out/bench_${tag}_$c.json 2> $out/bench_${tag}_$c.err; echo "bench $c=$?"
done
python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_${tag}_reference.json 2>&1; echo "reference=$?"
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --sustained-s 0 > $out/${tag}_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/${tag}_launches_bench.csv \
      python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --sustained-s 0 > $out/${tag}_ncu_launch.log 2>&1
echo "ncu launches=$?"
for c in C5 C2 C3 C4M; do
  python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-copy-ref --sustained-s 0 > $out/${tag}_plainf_$c.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:remap_tiled -s 3 -c 1 -o $out/${tag}_prof_$c \
        python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-copy-ref --sustained-s 0 > $out/${tag}_ncu_full_$c.log 2>&1
  echo "ncu full $c=$?"
  if [ -f $out/${tag}_prof_$c.ncu-rep ]; then
    ncu -i $out/${tag}_prof_$c.ncu-rep --page raw --csv > $out/${tag}_ncu_full_${c}_raw.csv 2>/dev/null
    ncu -i $out/${tag}_prof_$c.ncu-rep --page details --csv > $out/${tag}_ncu_full_${c}_details.csv 2>/dev/null
    rm -f $out/${tag}_prof_$c.ncu-rep
  fi
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none \
      -k regex:remap_tiled -s 4 -c 3 --csv --log-file $out/${tag}_steady_$c.csv \
      python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-copy-ref --sustained-s 0 > /dev/null 2>&1
  echo "steady $c=$?"
done
timeout 900 python tools/small_path_probe.py > $out/${tag}_small_path.log 2>&1; echo "small=$?"
python tools/b200_tuning_profile.py tests/golden/medical_b200_program.json $out/${tag}_b200_tuning_profile.json > $out/${tag}_b200_tuning_profile.log 2>&1; echo "tuning=$?"
for c in C2 C3 C4; do
  python bench.py --inplace --config $c > $out/bench_${tag}_inplace_$c.json 2> $out/bench_${tag}_inplace_$c.err; echo "inplace $c=$?"
done
du -sh $out
python tools/narrow_probe.py > $out/${tag}_narrow_probe.log 2>&1; echo "narrow=$?"
for i in 1 2; do ADHA_IP_TIMING=1 python tools/inplace_plan_time.py >> $out/${tag}_inplace_plan_time.log 2>&1; done; echo "plan=$?"
du -sh $out

#!/bin/bash
# GPU evidence for one round: parity tests, bench lines per config, launch list and one
# ncu --set full capture of the remap kernel per config (each ncu only after the same
# command exited 0 without ncu).  Outputs under gpurun_out/.
set -u
tag=${1:-r01}
out=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $out/pytest_gpu_$tag.log 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_$tag.log 2>&1; echo "smoke=$?"
python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench=$?"
for c in C1 C3 C3R C4 C5 P1 P2; do
  python bench.py --config $c --no-cpu-baseline > $out/bench_${tag}_$c.json 2> $out/bench_${tag}_$c.err; echo "bench $c=$?"
done
python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_${tag}_reference.json 2>&1; echo "reference=$?"
# launch list of the bench command (cold-cache, serialised: compare shares)
python bench.py --steps 2 --warmup 1 --soak-s 0 --no-cpu-baseline > $out/plain_$tag.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_$tag.csv \
      python bench.py --steps 2 --warmup 1 --soak-s 0 --no-cpu-baseline > $out/ncu_launch_$tag.log 2>&1
echo "ncu launches=$?"
for c in C2 C3 C3R C4 C5 P1 P2; do
  python bench.py --config $c --steps 2 --warmup 1 --soak-s 0 --no-cpu-baseline --no-e2e --no-copy-ref > $out/plainf_${tag}_$c.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:remap_tiled -s 3 -c 1 -o $out/prof_${tag}_$c \
        python bench.py --config $c --steps 2 --warmup 1 --soak-s 0 --no-cpu-baseline --no-e2e --no-copy-ref > $out/ncu_full_${tag}_$c.log 2>&1
  echo "ncu full $c=$?"
  # export on the box and drop the report: gpurun brings back at most 64 MiB
  if [ -f $out/prof_${tag}_$c.ncu-rep ]; then
    ncu -i $out/prof_${tag}_$c.ncu-rep --page raw --csv > $out/prof_${tag}_${c}_raw.csv 2>/dev/null
    ncu -i $out/prof_${tag}_$c.ncu-rep --page details --csv > $out/prof_${tag}_${c}_details.csv 2>/dev/null
    rm -f $out/prof_${tag}_$c.ncu-rep
  fi
done
# in-place remap (adha_remap_inplace): bench lines per config and one ncu --set full capture of
# C2's in-place kernels (each after the same command exited 0 without ncu)
for c in C2 C3 C3R C4 P1 P2; do
  python bench.py --inplace --config $c > $out/bench_${tag}_inplace_$c.json 2> $out/bench_${tag}_inplace_$c.err; echo "bench inplace $c=$?"
done
python tools/inplace_probe.py > $out/inplace_probe_$tag.log 2>&1; echo "inplace probe=$?"
python tools/inplace_probe.py --reps 2 --no-oop --cases C2 > $out/plain_ip_$tag.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ip_ -c 12 -o $out/prof_${tag}_inplace \
      python tools/inplace_probe.py --reps 2 --no-oop --cases C2 > $out/ncu_ip_$tag.log 2>&1
echo "ncu inplace=$?"
if [ -f $out/prof_${tag}_inplace.ncu-rep ]; then
  ncu -i $out/prof_${tag}_inplace.ncu-rep --page raw --csv > $out/prof_${tag}_inplace_raw.csv 2>/dev/null
  rm -f $out/prof_${tag}_inplace.ncu-rep
fi
du -sh $out

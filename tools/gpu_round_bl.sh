# round 2, call bl: ncu --set full and steady-state traffic of the final library for the configs
# the evidence runs do not capture (C3R, C4, P1, P2)
set -u
out=gpurun_out
tag=r02bl
for c in C3R C4 P1 P2; do
  ncu --set full --clock-control none --import-source on -k regex:remap_tiled -s 3 -c 1 -o $out/${tag}_prof_$c \
      python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-copy-ref --sustained-s 0 > $out/${tag}_ncu_full_$c.log 2>&1
  echo "ncu full $c=$?"
  if [ -f $out/${tag}_prof_$c.ncu-rep ]; then
    ncu -i $out/${tag}_prof_$c.ncu-rep --page raw --csv > $out/prof_${tag}_${c}_raw.csv 2>/dev/null
    ncu -i $out/${tag}_prof_$c.ncu-rep --page details --csv > $out/prof_${tag}_${c}_details.csv 2>/dev/null
    rm -f $out/${tag}_prof_$c.ncu-rep
  fi
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none \
      -k regex:remap_tiled -s 4 -c 3 --csv --log-file $out/${tag}_steady_$c.csv \
      python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-copy-ref --sustained-s 0 > /dev/null 2>&1
  echo "steady $c=$?"
done

# round 2, call c: byte-group shared-memory table A/B, where the tiled kernel's small-N time goes
set -u
out=gpurun_out
python tools/phase_probe.py --small > $out/c_phase_small.log 2>&1; echo "phase=$?"
timeout 600 python tools/small_path_probe.py > $out/c_small_path.log 2>&1; echo "small=$?"
for k in c3 g2; do
  python tools/one_remap.py $k 1 > $out/c_one_$k.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:remap_tiled -s 2 -c 1 -o $out/c_prof_$k \
      python tools/one_remap.py $k 1 > $out/c_ncu_$k.log 2>&1
  echo "ncu $k=$?"
  if [ -f $out/c_prof_$k.ncu-rep ]; then
    ncu -i $out/c_prof_$k.ncu-rep --page raw --csv > $out/c_prof_${k}_raw.csv 2>/dev/null
    ncu -i $out/c_prof_$k.ncu-rep --page source --csv --print-source cuda > $out/c_prof_${k}_src.csv 2>/dev/null
    ncu -i $out/c_prof_$k.ncu-rep --page details --csv > $out/c_prof_${k}_details.csv 2>/dev/null
  fi
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "byte or narrow or generalised or all_layout or config_shapes" > $out/c_pytest.log 2>&1; echo "pytest=$?"

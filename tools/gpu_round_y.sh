# round 2, call y: where does the C3-shape mid-size tiled launch spend its time? ncu --set full with
# source counters of the merged-plan kernel at 1 MB and 32 MB (tools/one_remap.py)
set -u
out=gpurun_out
python tools/one_remap.py c3 1 > $out/y_one.log 2>&1; echo "one=$?"
for mb in 1 32; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:remap_tiled -s 2 -c 1 \
    -o $out/y_c3_${mb}mb -f python tools/one_remap.py c3 $mb > $out/y_ncu_${mb}.log 2>&1; echo "ncu $mb=$?"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:remap_tiled -s 2 -c 1 \
    -o $out/y_c2_1mb -f python tools/one_remap.py c2 1 > $out/y_ncu_c2.log 2>&1; echo "ncu c2=$?"

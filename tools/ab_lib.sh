# Same-box A/B of product-library variants: each argument is a path to a libadha.so build
# (e.g. paper_1407_4859_b200/_build/old/libadha.so); "cur" is the in-tree library.  For each
# variant: the sustained C2 power probe and the burst ab_multi over narrow + chain edges.
set -u
cp paper_1407_4859_b200/libadha.so /tmp/libadha_cur.so
for round in 1 2; do
  for v in "$@"; do
    if [ "$v" = cur ]; then cp /tmp/libadha_cur.so paper_1407_4859_b200/libadha.so; else cp "$v" paper_1407_4859_b200/libadha.so; fi
    echo "== $v round $round"
    python tools/power_probe.py 3 2>&1 | grep "remap C2" | tail -1
    NARROW=1 CFGS=${CFGS:-C2,P1,P2,C4} ROUNDS=3 python tools/ab_multi.py "" 2>&1 | tail -14 | tr '\n' ' '; echo
  done
done
cp /tmp/libadha_cur.so paper_1407_4859_b200/libadha.so

cp paper_1407_4859_b200/libadha.so /tmp/cur.so
for r in 1 2; do for v in old cur; do
  if [ $v = old ]; then cp paper_1407_4859_b200/_build/old/libadha.so paper_1407_4859_b200/libadha.so; else cp /tmp/cur.so paper_1407_4859_b200/libadha.so; fi
  echo "== $v $r"; python tools/narrow_probe.py | tail -6 | sed -E 's/ +/ /g' | cut -c1-60 | tr '\n' ';'; echo; python tools/general_probe.py | tail -2 | cut -c1-60 | tr '\n' ';'; echo
done; done
cp /tmp/cur.so paper_1407_4859_b200/libadha.so

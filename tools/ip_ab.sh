#!/bin/bash
# A/B of compile-time variants of the in-place tile kernel: rebuild libadha.so with each
# define set, run the in-place probe, then restore the default build.
#   bash tools/ip_ab.sh "IP_LB=2" "IP_LB=4" "IP_LB=8"
set -u
cases=${CASES:-C2,P1,P2,C3s}
for v in "$@"; do
  python - "$v" <<'PY'
import sys, importlib.util
spec = importlib.util.spec_from_file_location("b", "paper_1407_4859_b200/build.py")
b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
defs = tuple(x for x in sys.argv[1].split() if x)
b.build(force=True, defines=defs, lib=b.LIB)
PY
  echo "== $v"
  python tools/inplace_probe.py --kernels --no-oop --cases $cases
done
python paper_1407_4859_b200/build.py --force > /dev/null

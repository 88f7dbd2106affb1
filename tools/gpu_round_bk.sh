# round 2, call bk: large randomised stress of the final library (2000 random out-of-place pairs,
# 1000 random in-place pairs with segment verification) and three default bench runs for the spread
set -u
out=gpurun_out
timeout 2400 python tools/stress_random.py 2000 4026 > $out/bk_stress_default.log 2>&1; echo "default=$?"
ADHA_IP_VERIFY=1 timeout 2400 python tools/stress_inplace.py 1000 4028 > $out/bk_stress_inplace.log 2>&1; echo "inplace=$?"
for i in 1 2 3; do python bench.py --no-cpu-baseline --no-e2e > $out/bk_bench_$i.json 2>/dev/null; done; echo "bench=$?"

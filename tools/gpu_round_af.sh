# round 2, call af: in-place host plan without the marking / cut-point passes; in-place GPU tests
set -u
out=gpurun_out
nproc > $out/af_plan_time.log
for i in 1 2; do ADHA_IP_TIMING=1 python tools/inplace_plan_time.py >> $out/af_plan_time.log 2>&1; done; echo "plan=$?"
ADHA_IP_VERIFY=1 timeout 1500 python -m pytest tests/test_gpu_inplace.py -m gpu -q -x > $out/af_pytest_inplace.log 2>&1; echo "pytest=$?"
python bench.py --inplace --config C3 --no-cpu-baseline --no-e2e > $out/af_bench_inplace_C3.json 2> $out/af_bench_inplace_C3.err; echo "bench=$?"

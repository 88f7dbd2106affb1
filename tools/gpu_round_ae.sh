# round 2, call ae: plan-table arena (no cudaMalloc under capture); loader / capture tests
set -u
out=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "capture" > $out/ae_pytest_capture.log 2>&1; echo "capture=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "loaders or write_back" > $out/ae_pytest.log 2>&1; echo "pytest=$?"

# round 2, call q: exact full-size checks everywhere
set -u
out=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > $out/q_pytest.log 2>&1; echo "pytest=$?"

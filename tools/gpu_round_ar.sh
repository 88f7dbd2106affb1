# round 2, call ar: randomised stress of the final library -- random layout pairs vs the oracle with
# the default loader rule and with the cp.async loader forced; random in-place pairs
set -u
out=gpurun_out
timeout 1200 python tools/stress_random.py 500 2026 > $out/ar_stress_default.log 2>&1; echo "default=$?"
ADHA_LOADER=cpa timeout 1200 python tools/stress_random.py 500 2027 > $out/ar_stress_cpa.log 2>&1; echo "cpa=$?"
ADHA_IP_VERIFY=1 timeout 1200 python tools/stress_inplace.py 300 2028 > $out/ar_stress_inplace.log 2>&1; echo "inplace=$?"

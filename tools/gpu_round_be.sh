# round 2, call be: randomised stress of the final library (PDL on) -- random layout pairs vs the oracle with
# the default loader rule and with the cp.async loader forced; random in-place pairs
set -u
out=gpurun_out
timeout 1200 python tools/stress_random.py 500 3026 > $out/be_stress_default.log 2>&1; echo "default=$?"
ADHA_LOADER=cpa timeout 1200 python tools/stress_random.py 500 3027 > $out/be_stress_cpa.log 2>&1; echo "cpa=$?"
ADHA_IP_VERIFY=1 timeout 1200 python tools/stress_inplace.py 300 3028 > $out/be_stress_inplace.log 2>&1; echo "inplace=$?"

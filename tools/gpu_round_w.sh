# round 2, call w: plain-copy patterns vs torch copy_ (tools/copy_probe.cu), 8 GiB per buffer
set -u
out=gpurun_out
python -c "
import torch
n=8<<30
a=torch.empty(n,dtype=torch.uint8,device='cuda').fill_(1); b=torch.empty_like(a)
for _ in range(3): b.copy_(a)
torch.cuda.synchronize()
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
for r in range(3):
  e0.record()
  for _ in range(10): b.copy_(a)
  e1.record(); torch.cuda.synchronize(); print('torch copy_ 8 GiB: %.0f GB/s' % (2*n*10/e0.elapsed_time(e1)/1e6))
" > $out/w_copy.log 2>&1
timeout 600 tools/copy_probe 8 >> $out/w_copy.log 2>&1; echo "probe=$?"

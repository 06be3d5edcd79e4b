#!/bin/bash
OUT=gpurun_out/${1:-s2p}
mkdir -p $OUT
for bk in 16 32; do for bn in 64 128 256; do
  for shp in "1024 1024 1024" "2048 2048 2048" "1024 1024 4096"; do
    set -- $shp
    ELV_TF32X3_BK=$bk ELV_TF32X3_BN=$bn timeout 120 python scripts/time_variant.py --variant parallel_tf32x3 --M $1 --N $2 --K $3 --reps 20 | sed "s/^{/{\"bk\": $bk, \"bn\": $bn, /" >> $OUT/sweep.jsonl 2>&1
  done
done; done
for bk in 16 32; do
  ELV_TF32X3_BK=$bk timeout 200 python -c "
import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2002_02268_b200 import interp, schedules, synth
M, N, K = 1000, 1100, 700
A = torch.empty((M, K), device='cuda'); B = torch.empty((K, N), device='cuda')
synth.fill_device(A, 4, 0); synth.fill_device(B, 4, 1)
t = schedules.apply_padded('parallel', M, N, K).term
np.save('$OUT/c$bk.npy', interp.run_tensor(t, A, B, tf32x3=True).cpu().numpy())
" >> $OUT/sweep.jsonl 2>&1
done
python -c "import numpy as np; a=np.load('$OUT/c16.npy'); b=np.load('$OUT/c32.npy'); print('bitwise_equal_bk16_bk32', np.array_equal(a,b))" >> $OUT/sweep.jsonl 2>&1
rm -f $OUT/c16.npy $OUT/c32.npy

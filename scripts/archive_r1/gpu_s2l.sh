#!/bin/bash
OUT=gpurun_out/${1:-s2l}
mkdir -p $OUT
for o in 2 3; do
  ELV_SGEMM_ORDER=$o timeout 200 python scripts/time_variant.py --variant parallel --n 8192 --reps 5 >> $OUT/order.jsonl 2>&1
  ELV_SGEMM_ORDER=$o timeout 200 python scripts/time_variant.py --variant parallel --M 32768 --N 32768 --K 8192 --reps 3 >> $OUT/order.jsonl 2>&1
done
for o in 2 3; do
  ELV_SGEMM_ORDER=$o timeout 200 python -c "
import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2002_02268_b200 import interp, schedules, synth
M, N, K = 2048, 4096, 1000
A = torch.empty((M, K), device='cuda'); B = torch.empty((K, N), device='cuda')
synth.fill_device(A, 4, 0); synth.fill_device(B, 4, 1)
t = schedules.apply_padded('parallel', M, N, K).term
np.save('$OUT/c$o.npy', interp.run_tensor(t, A, B).cpu().numpy())
" >> $OUT/order.jsonl 2>&1
done
python -c "import numpy as np; a=np.load('$OUT/c2.npy'); b=np.load('$OUT/c3.npy'); print('bitwise_equal', np.array_equal(a,b))" >> $OUT/order.jsonl 2>&1
rm -f $OUT/c2.npy $OUT/c3.npy
ELV_SGEMM_ORDER=3 timeout 600 python bench.py --variant parallel --steps 3 --no-cpu-baseline --no-e2e > $OUT/bench_simt_ffma2.json 2> $OUT/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k6_sgemm_ffma2 -s 1 -c 1 -o $OUT/prof_ffma2 \
  env ELV_SGEMM_ORDER=3 python scripts/profile_one.py --variant parallel --M 32768 --N 32768 --K 8192 --reps 2 > $OUT/prof.log 2>&1

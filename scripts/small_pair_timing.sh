#!/bin/bash
# small problems: the narrow CTA-pair kernel (ELV_SMALL_PAIR=64/128) vs the 1-CTA kernel -- call timing and bits
for sp in 0 64 128; do
  echo "ELV_SMALL_PAIR=$sp"
  ELV_SMALL_PAIR=$sp python scripts/small_timing_r2.py 2>&1 | grep -v '"parallel"'
  ELV_SMALL_PAIR=$sp python -c "
import hashlib, torch, sys
sys.path.insert(0, '.')
from paper_2002_02268_b200 import interp, schedules, synth
for n in (1024, 2048):
    A = torch.empty((n, n), device='cuda'); synth.fill_device(A, 0, 0)
    B = torch.empty((n, n), device='cuda'); synth.fill_device(B, 0, 1)
    t = schedules.apply('parallel', n, n, n).term
    for enc in ('tf32', 'fp16'):
        C = interp.run_tensor(t, A, B, tf32x3=True, tc_encoding=enc)
        print(n, enc, hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest()[:16])
"
done

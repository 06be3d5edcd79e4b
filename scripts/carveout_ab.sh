#!/bin/bash
# A/B of the max-shared-memory carveout preference (off by default) for the prepare / pack /
# fix-up kernels (ELV_PREP_CARVEOUT=0/1): small-call timing (1024^3, 2048^3)
# interleaved twice, then the default bench once each
OUT=gpurun_out/${1:-carveout}; mkdir -p $OUT
for r in 1 2; do for c in 0 1; do
  ELV_PREP_CARVEOUT=$c timeout 300 python scripts/small_timing_r2.py > $OUT/small_c${c}_$r.jsonl 2>&1
done; done
for c in 0 1; do
  ELV_PREP_CARVEOUT=$c timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ladder > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
done
for f in $OUT/small_*.jsonl; do echo $f; python -c "
import json
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print(d['n'], d['variant'], round(d['single_us'],1), round(d['b2b_us'],1))"; done
for f in $OUT/bench_c*.json; do python -c "
import json;d=json.load(open('$f'));r=d['roofline'];print('$f', round(d['value']/1e3,1), round(r['kernel_ms'],3), round(r['prepass_ms'],3), d['clocks']['sm_mhz'])"; done

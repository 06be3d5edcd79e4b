#!/bin/bash
OUT=gpurun_out/${1:-s2at}
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowshard.py -q --timeout 900 -p no:cacheprovider -k "fp16x3 or tf32x3 or bench_shape or checksums or 8192 or beyond or host or pipelined or strided" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
for i in 1 2; do
  timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $OUT/tma_$i.json 2> $OUT/tma_$i.err
  ELV_TMA_STORE_C=0 timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline > $OUT/reg_$i.json 2> $OUT/reg_$i.err
done
timeout 300 python scripts/k7_prof.py > $OUT/k7prof_fp16.jsonl 2>&1

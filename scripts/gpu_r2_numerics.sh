#!/bin/bash
# Round 2: chunked tcgen05 accumulation + range guard -- smoke, numerics tests, probe, quick bench
OUT=gpurun_out/${1:-r2_chunked}; mkdir -p $OUT
S=$OUT/summary.txt
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $S
tail -4 $OUT/smoke.log >> $S
timeout 1200 python -m pytest tests/test_gpu_numerics.py -q -s --timeout 600 -p no:cacheprovider > $OUT/numerics.log 2>&1; echo "numerics rc=$?" >> $S
tail -3 $OUT/numerics.log >> $S
timeout 600 python scripts/tc_numerics_r2.py > $OUT/tc_numerics.jsonl 2> $OUT/tc_numerics.err; echo "probe rc=$?" >> $S
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $S
timeout 600 python bench.py --variant parallel_tf32x3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_tf32.json 2> $OUT/bench_tf32.err; echo "bench tf32 rc=$?" >> $S

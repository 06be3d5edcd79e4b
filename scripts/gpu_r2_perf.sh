#!/bin/bash
# Round 2 tuning loop: cycle accounting (prof build) + short benches, both encodings
OUT=gpurun_out/${1:-r2_perf}; mkdir -p $OUT
S=$OUT/summary.txt
for enc in fp16 tf32; do
  ENC=$enc timeout 300 python scripts/k7_prof.py > $OUT/prof_$enc.jsonl 2>&1; echo "prof $enc rc=$?" >> $S
  tail -1 $OUT/prof_$enc.jsonl >> $S
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $S
timeout 600 python bench.py --variant parallel_tf32x3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_tf32.json 2> $OUT/bench_tf32.err; echo "bench tf32 rc=$?" >> $S
python scripts/bench_brief.py $OUT >> $S

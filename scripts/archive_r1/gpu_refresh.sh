#!/bin/bash
# Bench-line refresh (no ncu --set full captures): default bench, SIMT bench,
# ladder, reference arm, ncu launch list of the default bench command.
OUT=gpurun_out/${1:-refresh}
mkdir -p $OUT
S=$OUT/summary.txt
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $S
timeout 900 python bench.py --variant parallel --steps 3 --no-cpu-baseline > $OUT/bench_simt.json 2> $OUT/bench_simt.err; echo "bench simt rc=$?" >> $S
timeout 900 python bench.py --workload ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; echo "ladder rc=$?" >> $S
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "bench ref rc=$?" >> $S
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/launches_bench.log 2>&1; echo "launches rc=$?" >> $S
timeout 900 python bench.py > $OUT/bench2.json 2> $OUT/bench2.err; echo "bench2 rc=$?" >> $S

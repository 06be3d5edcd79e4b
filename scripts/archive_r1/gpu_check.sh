#!/bin/bash
# One gpurun call: smoke, GPU parity tests, ladder + default bench, launch list.
# Usage (from the build container):
#   gpurun --timeout 2400 -- bash scripts/gpu_check.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
echo "== smoke" | tee $OUT/summary.txt
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/summary.txt
tail -5 $OUT/smoke.log >> $OUT/summary.txt
echo "== pytest -m gpu" | tee -a $OUT/summary.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/summary.txt
tail -30 $OUT/pytest_gpu.log >> $OUT/summary.txt
echo "== ladder" | tee -a $OUT/summary.txt
timeout 600 python bench.py --workload ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; echo "ladder rc=$?" | tee -a $OUT/summary.txt
echo "== bench default" | tee -a $OUT/summary.txt
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" | tee -a $OUT/summary.txt
echo "== bench simt parallel" | tee -a $OUT/summary.txt
timeout 900 python bench.py --steps 3 --warmup 3 --variant parallel --no-e2e --no-cpu-baseline > $OUT/bench_simt.json 2> $OUT/bench_simt.err; echo "bench simt rc=$?" | tee -a $OUT/summary.txt

#!/bin/bash
# 3xFP16 prepare changes: fp16 GPU tests, prepare timing per mode, launch lists.
OUT=gpurun_out/${1:-fp}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -k "fp16 or warp_row or variant8 or 8-" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
timeout 600 python scripts/fp16_prep_timing.py > $OUT/prep.jsonl 2> $OUT/prep.err; echo "prep rc=$?" >> $OUT/summary.txt
timeout 600 python scripts/small_timing.py 1024 1024 1024 > $OUT/small1024.jsonl 2>&1; echo "small rc=$?" >> $OUT/summary.txt
timeout 600 python scripts/small_timing.py 2048 2048 2048 > $OUT/small2048.jsonl 2>&1; echo "small rc=$?" >> $OUT/summary.txt

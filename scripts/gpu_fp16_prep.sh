OUT=gpurun_out/fp1; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "fp16 or warp_row" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
timeout 600 python scripts/fp16_prep_timing.py > $OUT/prep.jsonl 2> $OUT/prep.err; echo "prep rc=$?" >> $OUT/summary.txt
ELV_FP16X3_WARP_ROWS=1 ELV_FP16X3_COLMAX_SLAB=64 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launch_old.csv python scripts/small_launches.py > /dev/null 2>&1; echo "ncu old rc=$?" >> $OUT/summary.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launch_new.csv python scripts/small_launches.py > /dev/null 2>&1; echo "ncu new rc=$?" >> $OUT/summary.txt

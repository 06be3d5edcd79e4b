#!/bin/bash
OUT=gpurun_out/${1:-s2by}
mkdir -p $OUT
for lib in libelevate_b200.so libelevate_b200_kt64.so; do
  ELV_LIB=$PWD/paper_2002_02268_b200/$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k16 --csv --log-file $OUT/k16_$lib.csv python scripts/profile_one.py --variant parallel_fp16x3 --M 32768 --N 32768 --K 8192 --reps 3 > $OUT/prof_$lib.log 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowshard.py -q -x -k "fp16 or host" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt

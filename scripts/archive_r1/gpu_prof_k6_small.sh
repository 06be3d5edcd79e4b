OUT=gpurun_out/k6s; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k6_sgemm_small -s 2 -c 1 -o $OUT/k6s_1024 \
  python scripts/profile_one.py --variant parallel --n 1024 --reps 4 > $OUT/k6s.log 2>&1; echo "rc=$?" >> $OUT/summary.txt

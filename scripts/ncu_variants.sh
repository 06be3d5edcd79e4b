#!/bin/bash
# Per-variant ncu counters (north star: FFMA throughput vs the SIMT peak per
# variant, tensor-pipe utilisation for 3xTF32, HBM GB/s for the packing
# kernels).  One capture per variant; the launch of interest is the last rep.
OUT=${1:-gpurun_out/ncu_variants}
mkdir -p $OUT
MET=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
for v in baseline blocking vectorized loopPerm arrayPacking cacheBlocks parallel parallel_tf32x3; do
  timeout 300 ncu --metrics $MET --clock-control none --csv --log-file $OUT/$v-1024.csv \
    python scripts/profile_one.py --variant $v --n 1024 --reps 3 > /dev/null 2>&1
done
for v in arrayPacking cacheBlocks parallel parallel_tf32x3; do
  timeout 600 ncu --metrics $MET --clock-control none --csv --log-file $OUT/$v-8192.csv -c 8 \
    python scripts/profile_one.py --variant $v --n 8192 --reps 2 > /dev/null 2>&1
done

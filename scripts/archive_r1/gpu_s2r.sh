#!/bin/bash
# the bench's N>1 path (PipelinedRowShardGemm, barriers, max-over-ranks) with 2 ranks sharing one GPU over gloo
OUT=gpurun_out/${1:-s2r}
mkdir -p $OUT
for v in parallel_tf32x3 parallel; do
ELV_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 \
  bench.py --gpus 2 --variant $v --M 4096 --N 4096 --K 2048 --steps 3 --warmup 3 > $OUT/bench2_$v.json 2> $OUT/bench2_$v.err; echo "bench2 $v rc=$?" >> $OUT/summary.txt
done
ELV_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 \
  bench.py --impl reference --gpus 2 --steps 1 --warmup 3 > $OUT/bench2_ref.json 2> $OUT/bench2_ref.err; echo "bench2 ref rc=$?" >> $OUT/summary.txt

"""Quick ladder subset for tuning runs: the tensor-core variants (and K6) at
1024^3 and a few small shapes, per-call GFLOP/s and kernel TFLOP/s (L2
flushed), through bench.ladder_cases' timing loop."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

bench.LADDER_1024 = ("parallel", "parallel_tf32x3", "parallel_fp16x3")
bench.LADDER_8192 = ("parallel_tf32x3", "parallel_fp16x3")
bench.ODD_SHAPES = ((2048, 2048, 2048), (1000, 1000, 1000), (4096, 256, 4096))
import torch  # noqa: E402

for r in bench.ladder_cases(torch.device("cuda", 0), reps_small=20, reps_large=5):
    print(json.dumps(r), flush=True)

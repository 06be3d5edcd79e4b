#!/bin/bash
# Session-2 first check: smoke, GPU tests (incl. generated kernels), PCIe probe, default bench.
OUT=gpurun_out/${1:-s2a}
mkdir -p $OUT
S=$OUT/summary.txt
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $S
timeout 120 python scripts/pcie_probe.py > $OUT/pcie.json 2>&1; echo "pcie rc=$?" >> $S
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S
tail -4 $OUT/pytest_gpu.log >> $S
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $S

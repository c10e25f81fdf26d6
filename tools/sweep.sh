#!/bin/bash
# BASELINE configs[4] sweep on one GPU: N in {3, 5, 7} x 8^3 .. 64^3 elements per GPU
# (TGV, affine, weak-scaling mesh builder), device-timed bench lines without the CPU
# arms -> gpurun_out/<tag>_sweep.jsonl.      tools/sweep.sh <tag>
TAG=${1:-sweep}
O=gpurun_out
mkdir -p $O
: > $O/${TAG}_sweep.jsonl
for N in 3 5 7; do
  for E in 8 16 32 64; do
    timeout 600 python bench.py --mesh tgv --degree $N --elems $E --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
      > $O/${TAG}_sweep_n${N}_e${E}.log 2>&1 && tail -1 $O/${TAG}_sweep_n${N}_e${E}.log >> $O/${TAG}_sweep.jsonl
  done
done
echo sweep-done

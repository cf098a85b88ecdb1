#!/usr/bin/env bash
# Forward split-threshold sweep (DSG_SPLIT_LEN) on one GPU: one rank of the
# N-GPU weak-scaling workload (tools/repro_rank.py) and the N=1 workload.
for sl in 0 16384 8192 4096; do
  for w in 4 1; do
    echo "== world $w rank 0 split $sl"
    DSG_SPLIT_LEN=$sl timeout 600 python tools/repro_rank.py --world $w --rank 0 --views 0 --train 20 2>&1 | grep -A12 "train ms"
  done
done

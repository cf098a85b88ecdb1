#!/usr/bin/env bash
# Segment / split threshold sweep (DSG_SEG_LEN, DSG_SPLIT_LEN) on one GPU:
# rank 0 of the N-GPU weak-scaling workload (tools/repro_rank.py).
W=${1:-4}
for cfg in "0 0" "0 8192" "0 4096"; do
  set -- $cfg
  echo "== world $W seg $1 split $2"
  DSG_SEG_LEN=$1 DSG_SPLIT_LEN=$2 timeout 600 python tools/repro_rank.py --world $W --rank 0 --views 0 --train 20 2>&1 | grep -A12 "train ms"
done

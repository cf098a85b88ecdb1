#!/usr/bin/env bash
# Work-unit sweeps on config 1 (sphere, 256²): DSG_SEG_LEN / DSG_SPLIT_LEN.
for cfg in "0 0"; do
  set -- $cfg
  DSG_SEG_LEN=$1 DSG_SPLIT_LEN=$2 python bench.py --workload sphere --res 256 --az 16 --el 4 --no-cpu-baseline --no-global > gpurun_out/seg_c1.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/seg_c1.json'));print('c1 seg $1 split $2', d['value'], d['stage_ms']['blend_fwd'], d['stage_ms']['blend_bwd'])"
done

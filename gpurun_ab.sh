#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
L=$PWD/paper_2509_12138_b200
show() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d.get('stage_ms'))" "$1"; }
for i in 1 2; do
  for v in base u2; do
    LIB=$L/libdsg_$v.so; [ $v = base ] && LIB=$L/libdsg.so
    DSG_LIB=$LIB timeout 600 python bench.py --no-cpu-baseline --no-global > gpurun_out/ab4_${v}_$i.json 2> gpurun_out/ab4_${v}_$i.err
    echo "$v $i rc=$?"; show gpurun_out/ab4_${v}_$i.json
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain --launch-skip 3 --launch-count 1 -o gpurun_out/chain_fused -f python bench.py --no-cpu-baseline --no-global --steps 2 --warmup 3 > gpurun_out/ab4_ncu.log 2>&1; echo ncu rc=$?

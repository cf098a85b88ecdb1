#!/usr/bin/env bash
# A/B of library variants on one B200: bench.py stage times, twice each,
# interleaved, then tools/ab_blend.py output differences against the first
# variant. Usage: bash tools/ab_round.sh base x y  (libdsg_<v>.so; "new" =
# libdsg.so). Results in gpurun_out/ab_*.
set -u
L=paper_2509_12138_b200
libof() { if [ "$1" = new ]; then echo "$PWD/$L/libdsg.so"; else echo "$PWD/$L/libdsg_$1.so"; fi; }
for i in 1 2; do for v in "$@"; do
  DSG_LIB=$(libof $v) timeout 600 python bench.py --no-cpu-baseline --no-global > gpurun_out/ab_${v}_$i.json 2> gpurun_out/ab_${v}_$i.err
  echo "$v $i rc=$?"; python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$i.json'));print(d['value'],d['ms_per_step'],d.get('stage_ms',''))"
done; done
for v in "$@"; do
  DSG_LIB=$(libof $v) timeout 600 python tools/ab_blend.py --out gpurun_out/ab_$v.npz > gpurun_out/ab_blend_$v.log 2>&1; echo "ab $v rc=$?"
done
for v in "${@:2}"; do
  python tools/ab_blend.py --compare gpurun_out/ab_$1.npz gpurun_out/ab_$v.npz > gpurun_out/ab_cmp_$v.log 2>&1
  echo "== $1 vs $v"; tail -15 gpurun_out/ab_cmp_$v.log
done
rm -f gpurun_out/ab_*.npz

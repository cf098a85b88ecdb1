#!/usr/bin/env bash
# Round-end measurement on one B200 (run through gpurun from the repo root):
# GPU parity tests, the bench line, the reference arm, the ncu launch list of
# the bench's timed steps and one ncu --set full capture of the step kernels.
# Outputs land in gpurun_out/<tag>_*; summaries are copied into profiles/.
set -u
tag=${1:-r01}
out=gpurun_out
mkdir -p "$out"
python -m pytest tests -m gpu -q > "$out/${tag}_pytest_gpu.log" 2>&1
tail -3 "$out/${tag}_pytest_gpu.log"
python bench.py > "$out/${tag}_bench.json" 2> "$out/${tag}_bench.err"
echo "bench rc=$?"; cat "$out/${tag}_bench.json"
python bench.py --impl reference > "$out/${tag}_bench_reference.json" 2> "$out/${tag}_bench_reference.err"
echo "reference rc=$?"; cat "$out/${tag}_bench_reference.json"
# launch list of the timed region only (NVTX range "dsg_timed" in bench.py)
ncu --nvtx --nvtx-include "dsg_timed/" --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file "$out/${tag}_launches.csv" \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-global \
    > "$out/${tag}_ncu_launch.log" 2>&1
echo "ncu launch rc=$?"
# full capture: one launch of each step kernel inside the timed region
ncu --nvtx --nvtx-include "dsg_timed/" --set full --clock-control none --import-source on \
    -k regex:"k_blend_bwd|k_blend_fwd|k_chain|k_adam|k_preprocess|k_onesweep|k_duplicate" -c 16 \
    -o "$out/${tag}_step_full" -f \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-global \
    > "$out/${tag}_ncu_full.log" 2>&1
echo "ncu full rc=$?"

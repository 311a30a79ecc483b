#!/bin/bash
# Sweep of the FMA-pipe exp2 share in the loss kernels (token_fact.cu
# ACCEL_F2_POLY_A / _C, ACCEL_GS2_POLY): rebuild with each define set, one
# cfg2 bench line each (K4 time = roofline.achieved's launch, step = ms_per_step).
set -u
out=${1:-gpurun_out/poly_sweep.jsonl}
: > "$out"
for v in "0 0 0" "1 1 1" "0 1 1" "1 0 0" "2 0 1" "1 1 0" "2 1 2"; do
  set -- $v
  export ACCEL_NVCC_DEFS="-DACCEL_F2_POLY_A=$1 -DACCEL_F2_POLY_C=$2 -DACCEL_GS2_POLY=$3"
  python -c "from paper_2603_18464_b200 import build; build.build()" 2>/dev/null || { echo "build failed $v"; continue; }
  line=$(python bench.py --steps 10 --warmup 3 --no-extra --no-cpu --no-e2e 2>/dev/null | tail -1)
  echo "{\"poly\": \"$v\", \"bench\": $line}" >> "$out"
  echo "$v: $(echo "$line" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"])')"
done
unset ACCEL_NVCC_DEFS
python -c "from paper_2603_18464_b200 import build; build.build()" 2>/dev/null

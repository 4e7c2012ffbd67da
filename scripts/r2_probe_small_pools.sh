#!/bin/bash
# Round-2 probe: C5 small-pool shapes (4x256) under different CTAs per SM and
# register budgets, then ncu captures (C3 bank conflicts, C4 launch list,
# worst C5 R=1 shape).  Run from the repo root on the GPU box.
cd ${GRAFT_REPO_ROOT:-/root/repo}
O=gpurun_out
mkdir -p $O
run() {  # lib pps only
  local lib=$1 pps=$2 only=$3
  WRNG_GPU_LIB=$PWD/paper_1004_3114_b200/$lib python scripts/sweep_c5.py --only $only \
    --pools-per-sm $pps --out $O/tmp_sweep.json 2>&1 | grep -E "^f(32|64)" | head -1 | sed "s/^/$lib pps=$pps: /"
}
for only in f32:256:1 f64:256:1; do
  for pps in 8 12 16; do run libwrng_gpu.so $pps $only; done
  run libwrng_gpu_oldminb.so 8 $only
done

#!/bin/bash
# A/B: the in-tree library vs a variant on the 4x256 C5 R=1 shapes, alternating.
cd ${GRAFT_REPO_ROOT:-/root/repo}
for rep in 1 2 3; do
  for lib in libwrng_gpu.so libwrng_gpu_$1.so; do
    for only in f32:256:1 f64:256:1; do
      WRNG_GPU_LIB=$PWD/paper_1004_3114_b200/$lib python scripts/sweep_c5.py --only $only \
        --out gpurun_out/tmp_sweep.json 2>&1 | grep -E "^f(32|64)" | head -1 | cut -c1-70 | sed "s/^/$lib: /"
    done
  done
done

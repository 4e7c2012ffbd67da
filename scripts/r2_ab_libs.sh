#!/bin/bash
# A/B of several library builds (same sources) on given C5 shapes, alternating.
# usage: r2_ab_libs.sh "lib1 lib2 ..." "f32:256:1 f64:256:1" [reps]
cd ${GRAFT_REPO_ROOT:-/root/repo}
for rep in $(seq ${3:-2}); do
  for lib in $1; do
    for only in $2; do
      WRNG_GPU_LIB=$PWD/paper_1004_3114_b200/$lib python scripts/sweep_c5.py --only $only \
        --out gpurun_out/tmp_sweep.json 2>&1 | grep -E "^f(32|64)" | head -1 | cut -c1-70 | sed "s/^/$lib: /"
    done
  done
done

#!/bin/bash
# Link-order A/B: C3 bench line and the 4x256 C5 shapes per library build,
# and the in-tree build with eager module loading.
cd ${GRAFT_REPO_ROOT:-/root/repo}
for rep in 1 2; do
for spec in libwrng_gpu.so libwrng_gpu_relink.so libwrng_gpu.so:EAGER; do
  lib=${spec%%:*}; envx=""
  [ "$spec" != "$lib" ] && envx="CUDA_MODULE_LOADING=EAGER"
  for only in f64:256:1 f32:256:1; do
    env $envx WRNG_GPU_LIB=$PWD/paper_1004_3114_b200/$lib python scripts/sweep_c5.py --only $only \
      --out gpurun_out/tmp_sweep.json 2>&1 | grep -E "^f(32|64)" | head -1 | cut -c1-70 | sed "s/^/$spec: /"
  done
  env $envx WRNG_GPU_LIB=$PWD/paper_1004_3114_b200/$lib python bench.py --config c3 --steps 5 --warmup 2 \
    --no-extras --no-cpu-baseline --e2e-steps 1 --e2e-sample 1048576 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$spec c3', round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"
done
done

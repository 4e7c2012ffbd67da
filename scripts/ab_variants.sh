# A/B timing of library variants on the C3 bench line (device-timed value).
# usage: bash scripts/ab_variants.sh "suffix1 suffix2 ..." [reps]
cd ${GRAFT_REPO_ROOT:-/root/repo}
vars=${1:-""}; reps=${2:-2}
for r in $(seq $reps); do
for v in $vars; do
  lib=libwrng_gpu.so; envx=""
  envx="WRNG_GPU_NO_BULK=1"
  case $v in base) envx="";; nobulk) ;; *) lib=libwrng_gpu_$v.so; envx="";; esac
  env $envx WRNG_GPU_LIB=$PWD/paper_1004_3114_b200/$lib timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --e2e-sample 1048576 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"
done; done

# A/B timing of library variants on the C3 bench line (device-timed value).
# usage: bash scripts/ab_variants.sh "spec1 spec2 ..." [reps] [extra bench args]
#   spec: base | name (uses paper_1004_3114_b200/libwrng_gpu_<name>.so)
#         | name:VAR=VALUE[,VAR=VALUE] (environment for the default library)
cd ${GRAFT_REPO_ROOT:-/root/repo}
specs=${1:-base}; reps=${2:-2}; extra=${3:-}
for r in $(seq $reps); do
for v in $specs; do
  lib=libwrng_gpu.so; envx=""
  case $v in
    base) ;;
    *:*) envx=$(echo ${v#*:} | tr ',' ' ');;
    *) lib=libwrng_gpu_$v.so;;
  esac
  env $envx WRNG_GPU_LIB=$PWD/paper_1004_3114_b200/$lib timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --e2e-sample 1048576 $extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('${v%%:*}', round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"
done; done

#!/bin/bash
# Round-2 probe: is C3's l1tex shared-load "bank conflict" count contention
# with the bulk-copy engine (which reads every emitted byte from shared
# memory)?  Metric-only ncu of the C3 fill with the bulk engine (default) and
# with warp-store emission (WRNG_GPU_NO_BULK=1); then run-to-run spread of the
# 4x256 C5 shapes.
cd ${GRAFT_REPO_ROOT:-/root/repo}
O=gpurun_out
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__sass_inst_executed_op_shared_ld.sum,smsp__sass_inst_executed_op_shared_st.sum,gpu__time_duration.sum,dram__bytes_write.sum
for v in bulk nobulk; do
  envx=""; [ $v = nobulk ] && envx="WRNG_GPU_NO_BULK=1"
  env $envx ncu --metrics $M --clock-control none -k regex:k_smem -s 1 -c 1 --csv \
    python scripts/c3_fill_once.py --total 1073741824 > $O/conflicts_$v.csv 2> $O/conflicts_$v.err
done
for rep in 1 2; do
  for only in f32:256:1 f64:256:1 f32:1024:1; do
    python scripts/sweep_c5.py --only $only --out $O/tmp_sweep.json 2>&1 | grep -E "^f(32|64)" | head -1
  done
done

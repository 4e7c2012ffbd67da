#!/bin/bash
# usage: ncu_capture.sh NAME CMD...  — one `ncu --set full --import-source on`
# capture of the first k_smem launch after the warm-up one, summarised on the
# box (the .ncu-rep is deleted: gpurun copies back at most 64 MiB).
cd ${GRAFT_REPO_ROOT:-/root/repo}
name=$1; shift
O=gpurun_out
ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-k_smem} -s ${SKIP:-1} -c 1 \
    -o $O/$name "$@" > $O/${name}_run.log 2>&1
python scripts/ncu_summary.py $O/$name.ncu-rep 30 > $O/${name}_summary.txt 2>&1
python scripts/ncu_bank_conflicts.py $O/$name.ncu-rep 1 > $O/${name}_bank_conflicts.txt 2>&1
ncu -i $O/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
ncu -i $O/$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>/dev/null
python scripts/ncu_sass.py $O/$name.ncu-rep ${SASS_MIN:-100000} > $O/${name}_sass.txt 2>&1
rm -f $O/$name.ncu-rep

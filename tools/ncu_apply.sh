# usage: bash tools/ncu_apply.sh <tag>
set -e
TAG=${1:-r1}
python tools/prof_apply.py C3 3 > gpurun_out/prof_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_sweep|k_reduced|k_inv_sparse}" -s ${KSKIP:-6} -c ${KCOUNT:-3} -o gpurun_out/prof_$TAG python tools/prof_apply.py C3 3 > gpurun_out/ncu_$TAG.log 2>&1
python tools/prof_apply.py C3 3 > gpurun_out/prof_plain2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_apply.py C3 3 > gpurun_out/ncu_launch_$TAG.log 2>&1

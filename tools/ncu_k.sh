# usage: bash tools/ncu_k.sh <cfg> <kernel-regex> <skip> <tag>
CFG=$1; KR=$2; SK=$3; TAG=$4
PYTHONPATH=. python tools/prof_apply.py $CFG 2 > gpurun_out/plain_$TAG.log 2>&1 && PYTHONPATH=. ncu --set full --clock-control none --import-source on -k regex:"$KR" -s $SK -c 1 -o gpurun_out/prof_$TAG python tools/prof_apply.py $CFG 2 > gpurun_out/ncu_$TAG.log 2>&1

# usage: bash tools/ncu_kd.sh <cfg> <demangled-kernel-regex> <skip> <tag>   (full set, one launch)
CFG=$1; KR=$2; SK=$3; TAG=$4
PYTHONPATH=. python tools/prof_apply.py $CFG 2 > gpurun_out/plain_$TAG.log 2>&1 && PYTHONPATH=. ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$KR" -s $SK -c 1 -o gpurun_out/prof_$TAG python tools/prof_apply.py $CFG 2 > gpurun_out/ncu_$TAG.log 2>&1

# usage: bash tools/ncu_solve.sh <cfg> <demangled-kernel-regex> <skip> <count> <tag>  (ncu --set full on solve launches)
CFG=$1; KR=$2; SK=$3; CN=$4; TAG=$5
PYTHONPATH=. python tools/prof_solve.py $CFG 2 > gpurun_out/plain_$TAG.log 2>&1 && PYTHONPATH=. ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$KR" -s $SK -c $CN -o gpurun_out/prof_$TAG python tools/prof_solve.py $CFG 2 > gpurun_out/ncu_$TAG.log 2>&1

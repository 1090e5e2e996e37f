# usage: bash tools/ncu_launch.sh <cfg> <tag>
CFG=${1:-C3}; TAG=${2:-x}
PYTHONPATH=. python tools/prof_apply.py $CFG 2 > gpurun_out/plain_$TAG.log 2>&1 && PYTHONPATH=. ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_apply.py $CFG 2 > gpurun_out/ncu_launch_$TAG.log 2>&1

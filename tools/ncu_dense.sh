set -e
TAG=${1:-d1}
PYTHONPATH=. python tools/prof_dense.py C3 > gpurun_out/dense_plain.log 2>&1
PYTHONPATH=. ncu --set full --clock-control none --import-source on -k regex:"k_dst_dense" -s 4 -c 2 -o gpurun_out/prof_$TAG python tools/prof_dense.py C3 > gpurun_out/ncu_$TAG.log 2>&1

# ncu launch list of two C3 solves (dense / final-field kernels)
PYTHONPATH=. ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/solve_launches.csv python tools/prof_solve.py C3 2 > gpurun_out/ncu_sl.log 2>&1

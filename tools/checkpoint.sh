# Full GPU checkpoint: tests, bench lines (C3 default, C5), launch lists, full ncu of the top kernels.
set -x
mkdir -p gpurun_out/ck
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/ck/tests.log 2>&1
tail -3 gpurun_out/ck/tests.log
timeout 600 python bench.py > gpurun_out/ck/bench_C3.json 2> gpurun_out/ck/bench_C3.err
timeout 900 python bench.py --config C5 --no-cpu-baseline > gpurun_out/ck/bench_C5.json 2> gpurun_out/ck/bench_C5.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/ck/bench_ref.json 2> gpurun_out/ck/bench_ref.err
PYTHONPATH=. ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/ck/launches_C3_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ck/ncu_bench.log 2>&1
bash tools/ncu_launch.sh C3 ckC3 > /dev/null 2>&1; mv gpurun_out/launches_ckC3.csv gpurun_out/ck/launches_C3_apply.csv
bash tools/ncu_launch.sh C5 ckC5 > /dev/null 2>&1; mv gpurun_out/launches_ckC5.csv gpurun_out/ck/launches_C5_apply.csv
bash tools/ncu_kd.sh C3 "k_inv_sparse" 0 ckinv; mv gpurun_out/prof_ckinv.ncu-rep gpurun_out/ck/
bash tools/ncu_kd.sh C3 "k_sweep<\(int\)0>" 0 cksw; mv gpurun_out/prof_cksw.ncu-rep gpurun_out/ck/
bash tools/ncu_kd.sh C5 "k_fwd3s" 0 ckfwd; mv gpurun_out/prof_ckfwd.ncu-rep gpurun_out/ck/
bash tools/ncu_kd.sh C5 "k_inv3y" 0 ckinv3; mv gpurun_out/prof_ckinv3.ncu-rep gpurun_out/ck/
timeout 600 python bench.py --config C2 --bc neumann --no-cpu-baseline > gpurun_out/ck/bench_C2N.json 2> gpurun_out/ck/bench_C2N.err
python tools/setup_timing.py > gpurun_out/ck/setup_timing.jsonl 2>&1
python tools/setup_timing.py --config C2 --n 8192 >> gpurun_out/ck/setup_timing.jsonl 2>&1

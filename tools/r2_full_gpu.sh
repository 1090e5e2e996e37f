# the whole -m gpu suite (incl. the full-size tests) and smoke(), as the round-end driver runs them
export PYTHONPATH=.
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2_gputests_all.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2_gputests_all.log
tail -n 3 gpurun_out/r2_gputests_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
tail -n 3 gpurun_out/r2_smoke.log

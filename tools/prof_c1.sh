export PYTHONPATH=.
for r in 1 2 3; do python tools/prof_apply.py C1 3 2>&1 | tail -n 1; done
python tools/prof_apply.py C2 3 2>&1 | tail -n 1

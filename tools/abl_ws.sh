export PYTHONPATH=.
for a in 0 1 2; do echo "ws abl=$a"; KFBI_WS_ABL=$a python tools/prof_apply.py C3 3 2>&1 | tail -1; done
for a in 0 1 2; do echo "old abl=$a"; KFBI_WS_ABL=$a KFBI_INV_OLD=1 python tools/prof_apply.py C3 3 2>&1 | tail -1; done

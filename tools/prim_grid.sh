export PYTHONPATH=$PWD
for g in 4 16 48 98 148 296; do echo "grid $g"; DMST_PRIM_GRID=$g timeout 120 python tools/mreach_time.py 100000 | tail -1; done

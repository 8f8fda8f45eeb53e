timeout -s KILL 300 python tools/e2e_prof.py 10000 2>&1 | tail -4
timeout -s KILL 300 python tools/e2e_prof.py 10000 12 2>&1 | tail -2
timeout -s KILL 300 python tools/e2e_prof.py 10000 48 2>&1 | tail -2

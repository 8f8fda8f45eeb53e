# deep-ramp under synccheck / racecheck: graph vs eager, default vs more tracked barriers
S=/usr/local/cuda/bin/compute-sanitizer
O=gpurun_out/san19.log; : > $O
timeout -s KILL 600 python tools/sanitize_run.py deep-ramp >> $O 2>&1; echo "plain deep-ramp rc=$?" >> $O
timeout -s KILL 600 $S --tool synccheck --error-exitcode 9 python tools/sanitize_run.py deep-ramp >> $O 2>&1; echo "synccheck graph rc=$?" >> $O
SAN_EAGER=1 timeout -s KILL 600 $S --tool synccheck --error-exitcode 9 python tools/sanitize_run.py deep-ramp >> $O 2>&1; echo "synccheck eager rc=$?" >> $O
timeout -s KILL 600 $S --tool synccheck --num-cuda-barriers 4096 --error-exitcode 9 python tools/sanitize_run.py deep-ramp >> $O 2>&1; echo "synccheck graph nb4096 rc=$?" >> $O
SAN_EAGER=1 timeout -s KILL 600 $S --tool racecheck --error-exitcode 9 python tools/sanitize_run.py deep-ramp >> $O 2>&1; echo "racecheck eager rc=$?" >> $O
SAN_EAGER=1 timeout -s KILL 600 $S --tool racecheck --num-cuda-barriers 4096 --error-exitcode 9 python tools/sanitize_run.py deep-ramp >> $O 2>&1; echo "racecheck eager nb4096 rc=$?" >> $O

#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (each schedule case in its own
# process); logs to gpurun_out/sanitize_<tool>.log, one summary line per case.
cases=${CASES:-$(python tools/sanitize_run.py list)}
tag=${TAG:-}
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  log=gpurun_out/sanitize${tag}_$tool.log; : > $log
  for c in $cases; do
    timeout -s KILL 600 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 10 --error-exitcode 9 \
      $( [ $tool = memcheck ] && echo --leak-check full ) python tools/sanitize_run.py $c >> $log 2>&1
    echo "$tool $c rc=$?" | tee -a $log
  done
done

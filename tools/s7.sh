CASES='tiles all-escape half-escape all-escape-coop n2 mfd forest' TAG=_r02g TOOLS='memcheck synccheck initcheck' bash tools/sanitize.sh > /dev/null 2>&1
CASES='tiles all-escape half-escape n2 mfd' TAG=_r02g_eager TOOLS='racecheck' SAN_EAGER=1 bash tools/sanitize.sh > /dev/null 2>&1
grep -h "rc=" gpurun_out/sanitize_r02g_*.log

timeout -s KILL 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity_large.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1
CASES="tiles half-escape all-escape n2" TOOLS="memcheck racecheck" TAG=_r02j bash tools/sanitize.sh 2>&1 | grep "rc="

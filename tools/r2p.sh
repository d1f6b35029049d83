set -u
O=gpurun_out/r2p; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize_cases.py > $O/memcheck.log 2>&1; echo "memcheck rc=$?"
timeout 1500 $CS --tool racecheck --racecheck-report analysis --error-exitcode 9 python tools/sanitize_cases.py C2 C5 > $O/racecheck.log 2>&1; echo "racecheck rc=$?"
timeout 1200 $CS --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py C2 C5 > $O/synccheck.log 2>&1; echo "synccheck rc=$?"

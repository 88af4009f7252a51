#!/bin/bash
cd "$(dirname "$0")/.."
D=gpurun_out/r02s; mkdir -p $D
timeout -s KILL 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > $D/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 $D/memcheck.log
timeout -s KILL 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_small.py > $D/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 $D/racecheck.log

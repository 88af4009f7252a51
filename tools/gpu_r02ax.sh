#!/bin/bash
# compute-sanitizer over every kernel path on the final build
cd /root/repo
D=gpurun_out/r02ax; mkdir -p $D
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > $D/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -2 $D/memcheck.log
timeout -s KILL 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_small.py > $D/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -2 $D/racecheck.log
timeout -s KILL 1200 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_small.py > $D/synccheck.log 2>&1; echo "synccheck rc=$?"; tail -2 $D/synccheck.log

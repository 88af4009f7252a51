#!/bin/bash
# racecheck after the per-half exponent copies in gtp_grid_tc; L = 10 / 11 timing (KH = 88 variant)
cd /root/repo
D=gpurun_out/r02w; mkdir -p $D
timeout 300 python tools/grid_quad_timing.py 10,11 auto gtp_grid > $D/tc_l11.jsonl 2>&1; cat $D/tc_l11.jsonl
timeout 300 python tools/grid_quad_timing.py 10,11 auto gtp_fourier >> $D/tc_l11.jsonl 2>&1; tail -2 $D/tc_l11.jsonl
timeout -s KILL 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 400 python tools/sanitize_small.py > $D/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 $D/racecheck.log
grep -h "Write Thread\|Read Thread" $D/racecheck.log | grep -o "tpo_b200::<unnamed>::[a-z_0-9]*kernel" | sort | uniq -c
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -q -x -k "tcgen05 or degree_groups or weighted" 2>&1 | tail -2

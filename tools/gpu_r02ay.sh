#!/bin/bash
cd /root/repo
D=gpurun_out/r02ay; mkdir -p $D
timeout -s KILL 1200 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_small.py > $D/synccheck.log 2>&1; echo "synccheck rc=$?"; tail -2 $D/synccheck.log
grep "Device Frame" $D/synccheck.log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | sort -rn | head -5
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py tests/test_gpu_backward.py -k mtp -x -q 2>&1 | tail -1
timeout 300 python tools/grid_small_paths.py 2>/dev/null | head -0

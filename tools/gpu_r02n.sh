#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02n
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cgtp_bwd -c 2 -s 4 -o gpurun_out/r02n/bwd_tc python tools/profile_cgtp_bwd.py 6 > gpurun_out/r02n/ncu.log 2>&1
tail -3 gpurun_out/r02n/ncu.log

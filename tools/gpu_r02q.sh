#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02q
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mtp_kernel -c 1 -s 2 -o gpurun_out/r02q/mtp_L7b python tools/profile_mtp.py 7 > gpurun_out/r02q/ncu7.log 2>&1

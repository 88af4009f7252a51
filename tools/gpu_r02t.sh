#!/bin/bash
cd "$(dirname "$0")/.."
LS="4 6 10 12" bash tools/cgtp_prof.sh
timeout 300 python tools/bwd_timing.py --kinds cgtp --Ls 4,6,8,10,12 --batch 16384

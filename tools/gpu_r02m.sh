#!/bin/bash
cd "$(dirname "$0")/.."
for d in 0 1 2 4 6 7; do echo "== dbg $d"; TPO_CGTP_BWD_DBG=$d timeout 120 python tools/bwd_timing.py --kinds cgtp --Ls 3,6; done

#!/bin/bash
cd "$(dirname "$0")/.."
for d in 0 1 2 4 3 5 6 7; do echo "== dbg $d"; TPO_CGTP_DBG=$d timeout 120 python tools/cgtp_paths.py 4,6,8 2>&1 | grep -v Warn; done

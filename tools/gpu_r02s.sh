#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/ -x -q -m gpu -k "mtp" 2>&1 | tail -3
for d in 0 1 4; do echo "== dbg $d"; TPO_MTP_DBG=$d timeout 300 python tools/mtp_simt_timing.py; done

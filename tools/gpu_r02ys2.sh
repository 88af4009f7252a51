#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/ -x -q -m gpu -k "cgtp" 2>&1 | tail -2
for lib in head new head new; do echo "== $lib"; TPO_LIB_PATH=tools/ab/libtpo_$lib.so timeout 600 python tools/cgtp_paths.py 4,6,8,10,12,14,16; done

#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/ -x -q -m gpu -k "cgtp" 2>&1 | tail -3
for lib in base new base new; do echo "== $lib"; TPO_LIB_PATH=tools/ab/libtpo_$lib.so timeout 300 python tools/cgtp_paths.py 4,5,6,8,10,12; done

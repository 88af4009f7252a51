#!/bin/bash
cd "$(dirname "$0")/.."
echo "== yseg all"; TPO_CGTP_YSEG_MIN=16 timeout 600 python tools/cgtp_paths.py 6,8,9,10,11,12
echo "== row"; TPO_CGTP_YSEG_MIN=100000 timeout 600 python tools/cgtp_paths.py 6,8,9,10,11,12

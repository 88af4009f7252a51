#!/bin/bash
cd "$(dirname "$0")/.."
echo "== tc"; timeout 600 python tools/cgtp_paths.py
echo "== simt"; TPO_CGTP_TC=0 timeout 900 python tools/cgtp_paths.py

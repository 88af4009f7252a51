#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/ -x -q -m gpu -k "mtp" 2>&1 | tail -3
timeout 300 python tools/mtp_simt_timing.py

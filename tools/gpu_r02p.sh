#!/bin/bash
cd "$(dirname "$0")/.."
TPO_CGTP_BWD_PROF=1 timeout 120 python tools/profile_cgtp_bwd.py 6 2>&1 | tail -1

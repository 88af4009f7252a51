#!/bin/bash
cd "$(dirname "$0")/.."
for i in 1 2; do TPO_VERBOSE=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cgtp_bwd_tc --csv python tools/profile_cgtp_bwd.py 6 2>&1 | grep -o '"gpu__time_duration.sum","[^"]*","[^"]*"\|cgtp bwd tcgen05.*' | tail -2; done

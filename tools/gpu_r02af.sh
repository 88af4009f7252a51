#!/bin/bash
cd /root/repo
for L in 6 9 10 12 14 16; do
  B=65536; [ $L -ge 14 ] && B=16384
  TPO_CGTP_PROF=1 timeout -s KILL 120 python tools/profile_kernel.py --kind cgtp --L $L --batch $B --reps 2 2>&1 | grep -E "tpo-prof" | tail -1 | sed "s/^/L=$L /"
done

#!/bin/bash
# build the CUDA library in-tree; fail loudly; report spills
set -e
make -s -j8 -C /root/repo/paper_2506_13523_b200/csrc 2>&1 | grep -E "error|warning: v" || true
test -f /root/repo/paper_2506_13523_b200/libtpo_b200.so
for f in /root/repo/paper_2506_13523_b200/csrc/build/kernels/*.o.log; do
  n=$(grep -cE "[1-9][0-9]* bytes spill" "$f" || true); [ "$n" != "0" ] && echo "SPILLS in $f"
done
find /root/repo/paper_2506_13523_b200/csrc -path "*/csrc/tools" -prune -o -newer /root/repo/paper_2506_13523_b200/libtpo_b200.so -name "*.c*" -print -o -newer /root/repo/paper_2506_13523_b200/libtpo_b200.so -name "*.h*" -print | grep . && { echo "STALE BUILD"; exit 1; }
echo "build ok $(date +%T)"

#!/bin/bash
# MTP tcgen05: row halves meet on an mbarrier instead of a named barrier; synccheck, parity, timing A/B
cd /root/repo
P=paper_2506_13523_b200/libtpo_b200.so
cp $P /tmp/lib_new.so
for V in old new old new; do
  if [ $V = old ]; then cp lib_mtpold.so.tmp $P; else cp /tmp/lib_new.so $P; fi
  echo "== $V"; timeout 300 python tools/grid_quad_timing.py 2,4,5,6 auto mtp 2>/dev/null | cut -c1-80
done
cp /tmp/lib_new.so $P
timeout -s KILL 1200 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/synccheck_mbar.log 2>&1; echo "synccheck rc=$?"; tail -1 gpurun_out/synccheck_mbar.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py tests/test_gpu_backward.py tests/test_gpu_stages.py -k "mtp" -x -q 2>&1 | tail -1

#!/bin/bash
# A/B: mbarrier try_wait suspend hint (libtpo_hint) vs base, per kind and L
cd "$(dirname "$0")/.."
for lib in base hint base hint; do echo "== $lib"; TPO_LIB_PATH=tools/ab/libtpo_$lib.so timeout 300 python tools/kind_timing.py 2>&1 | tail -40 > gpurun_out/r02u_$lib.txt; cat gpurun_out/r02u_$lib.txt | tr '\n' ' ' | head -c 3000; echo; done

#!/bin/bash
cd "$(dirname "$0")/.."
for lib in pipe3 pipe5 pipe3 pipe5; do for ck in 16384 32768; do TPO_LIB_PATH=tools/ab/libtpo_$lib.so TPO_HOST_CHUNK_KB=$ck timeout 120 python tools/e2e_batch.py | sed "s/^/$lib /"; done; done

#!/bin/bash
cd "$(dirname "$0")/.."
for ck in 16384 32768 65536 131072; do for o in desc asc; do E2E_ORDER=$o TPO_HOST_CHUNK_KB=$ck timeout 120 python tools/e2e_batch.py; done; done

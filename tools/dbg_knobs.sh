#!/bin/bash
# forward time with parts of the U-Net pipeline disabled (PS_TC_DBG bits: 1 epilogue math,
# 2 MMAs, 8 activation loads, 16 weight loads) -> which stage is the critical path
cd "$(dirname "$0")/.."
for d in ${DBGS:-0 1 2 3 8 24 25 26 27}; do
  echo -n "dbg=$d "; PS_TC_DBG=$d timeout 120 python tools/time_fwd.py 1024 2>&1 | tail -1
done
echo -n "no_resident "; PS_NO_RESIDENT=1 timeout 120 python tools/time_fwd.py 1024 2>&1 | tail -1
echo -n "no_pdl "; PS_NO_PDL=1 timeout 120 python tools/time_fwd.py 1024 2>&1 | tail -1

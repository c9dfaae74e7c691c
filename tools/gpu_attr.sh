#!/bin/bash
# per-layer U-Net launch times (ncu gpu__time_duration, one forward at 1024 x 32) for PS_TC_DBG values
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for d in ${DBGS:-0 32}; do
  PS_TC_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:unet_tc_kernel \
     --log-file gpurun_out/attr_$d.csv python tools/profile_unet.py 1024 2 > /dev/null 2>&1
  echo "dbg=$d rc=$?"
done

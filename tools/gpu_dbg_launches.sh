#!/bin/bash
# one-forward launch lists with parts of the pipeline disabled (PS_TC_DBG bits)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
U="python tools/profile_unet.py 1024 1"
for d in ${DBGS:-1 2 24}; do
  PS_TC_DBG=$d timeout 300 $U > gpurun_out/unet_plain_$d.log 2>&1 && \
  PS_TC_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fwd_launches_dbg$d.csv $U > gpurun_out/ncu_dbg$d.log 2>&1
  echo "dbg $d rc=$?"
done

#!/bin/bash
# one-forward launch lists with and without an env knob (A/B per layer)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
U="python tools/profile_unet.py 1024 1"
timeout 300 $U > gpurun_out/unet_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fwd_launches.csv $U > /dev/null 2>&1
echo "A rc=$?"
env $KNOB timeout 300 $U > gpurun_out/unet_plain_b.log 2>&1 && \
  env $KNOB timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fwd_launches_b.csv $U > /dev/null 2>&1
echo "B rc=$?"

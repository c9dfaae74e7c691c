#!/bin/bash
# ncu --set full of one U-Net forward (all 29 unet_tc_kernel launches) at 1024 problems x 32 seeds
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
U="python tools/profile_unet.py ${P:-1024} 1"
$U > gpurun_out/unet_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"unet_tc|im2col|film_step" -c 31 -o gpurun_out/prof_unet -f $U > gpurun_out/ncu_unet.log 2>&1
echo "unet ncu rc=$?"
tail -3 gpurun_out/ncu_unet.log

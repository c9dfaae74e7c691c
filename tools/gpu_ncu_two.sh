#!/bin/bash
# ncu --set full of two U-Net layers of one forward (unet launch indices SKIP_A, SKIP_B)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
U="python tools/profile_unet.py 1024 1"
$U > gpurun_out/unet_plain.log 2>&1 || exit 1
for s in ${SKIPS:-2 12}; do
  ncu --set full --clock-control none --import-source on -k regex:unet_tc --launch-skip $s --launch-count 1 \
      -o gpurun_out/prof_l$s -f $U > gpurun_out/ncu_l$s.log 2>&1
  echo "layer $s rc=$?"
done

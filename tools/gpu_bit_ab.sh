#!/bin/bash
# bitwise comparison of the layered sampler between the working build and BASE (a .so path),
# then the quick A/B (tools/gpu_ab_quick.sh)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
timeout 600 python tools/dump_sample.py gpurun_out/ab/head.npz > /dev/null 2>&1
PS_LIB_OVERRIDE=$PWD/$BASE timeout 600 python tools/dump_sample.py gpurun_out/ab/base.npz > /dev/null 2>&1
python tools/bitcmp.py gpurun_out/ab/head.npz gpurun_out/ab/base.npz; echo "bitcmp rc=$?"; rm -f gpurun_out/ab/*.npz
LIBS="base=$BASE" bash tools/gpu_ab_quick.sh

#!/bin/bash
# bitwise + throughput A/B of the working build against abtmp/libps_old.so
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
python tools/dump_sample.py /tmp/ab_new.npz > gpurun_out/ab/dump_new.log 2>&1
PS_LIB_OVERRIDE=$PWD/${OLDLIB:-abtmp/libps_old.so} python tools/dump_sample.py /tmp/ab_old.npz > gpurun_out/ab/dump_old.log 2>&1
python tools/bitcmp.py /tmp/ab_old.npz /tmp/ab_new.npz > gpurun_out/ab/bitcmp.log 2>&1
cat gpurun_out/ab/dump_new.log gpurun_out/ab/bitcmp.log
timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_sampler_gpu.py -m gpu -x -q 2>&1 | tail -3
ROUNDS=${ROUNDS:-2} LIBS="${LIBS:-old=abtmp/libps_old.so}" bash tools/ab_multi.sh 2>&1 | tee gpurun_out/ab/ab.log

#!/bin/bash
# quick GPU check after a U-Net change: tc/sampler tests, forward timing, one-forward launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tc_gpu.py tests/test_sampler_gpu.py ${EXTRA_TESTS} -x -q > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_quick.log
timeout 300 python tools/time_fwd.py 1024 > gpurun_out/time_fwd.json 2>&1; echo "time_fwd rc=$?"; cat gpurun_out/time_fwd.json
if [ "${NCU:-1}" = 1 ]; then
U="python tools/profile_unet.py 1024 1"
timeout 300 $U > gpurun_out/unet_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fwd_launches.csv $U > gpurun_out/ncu_fwd.log 2>&1
echo "launch list rc=$?"
fi

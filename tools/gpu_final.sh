#!/bin/bash
# end-of-round evidence in one gpurun call: GPU tests, bench line, bench launch list, ncu --set full
# of one U-Net forward, persistent-sampler trace, config-4 sweep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/bench_small.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
P=1024 timeout 1500 bash tools/gpu_ncu_unet.sh
PS_NO_GRAPH=1 PS_PERSIST=1 PS_PERSIST_TRACE=gpurun_out/trace_final.bin timeout 300 python tools/persist_trace.py --run 1 32 && python tools/persist_trace.py gpurun_out/trace_final.bin 50 > gpurun_out/persist_trace.txt; echo "trace rc=$?"
timeout 1800 python tools/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"

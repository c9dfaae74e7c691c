#!/bin/bash
# One gpurun call: GPU tests, the default bench line, the bench launch list and ncu --set full
# captures of the U-Net convs and the refinement/ESDF kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json
[ "${SKIP_NCU:-0}" = 1 ] && exit 0
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/bench_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
U="python tools/profile_unet.py 1024 1"
$U > gpurun_out/unet_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:conv_tc -o gpurun_out/prof_unet -f $U > gpurun_out/ncu_unet.log 2>&1
echo "unet ncu rc=$?"
R="python tools/time_refine.py"
$R > gpurun_out/refine_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"bl_refine|esdf" -c 4 -o gpurun_out/prof_refine -f $R > gpurun_out/ncu_refine.log 2>&1
echo "refine ncu rc=$?"
cat gpurun_out/refine_plain.log

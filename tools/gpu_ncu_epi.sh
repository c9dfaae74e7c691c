#!/bin/bash
# ncu --set full (source-level) of the final layer and of one level-0 GN/FiLM layer inside the
# DDPM sampler at 1024 x 32 (PS_NO_GRAPH: plain launches)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PS_NO_GRAPH=1
python tools/profile_sample.py 1024 > gpurun_out/ps_plain.log 2>&1 || exit 1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
$NCU -k regex:"\(int\)64, \(int\)3" --launch-skip 5 -c 1 -o gpurun_out/prof_fin -f python tools/profile_sample.py 1024 > gpurun_out/ncu_fin.log 2>&1
echo "fin rc=$?"
$NCU -k regex:"\(int\)64, \(int\)1, \(bool\)0, \(int\)2, \(bool\)0" --launch-skip 4 -c 1 -o gpurun_out/prof_l0 -f python tools/profile_sample.py 1024 > gpurun_out/ncu_l0.log 2>&1
echo "l0 rc=$?"
tail -2 gpurun_out/ncu_l0.log

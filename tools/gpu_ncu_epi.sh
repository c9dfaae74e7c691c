#!/bin/bash
# ncu --set full (source-level) of single layers inside the DDPM sampler at 1024 x 32
# (PS_NO_GRAPH: plain launches).  KSEL="name:regex:skip|name:regex:skip" picks the layers.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PS_NO_GRAPH=1
python tools/profile_sample.py 1024 > gpurun_out/ps_plain.log 2>&1 || exit 1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
IFS='|' read -ra SPECS <<< "${KSEL:-fin:\(int\)64, \(int\)3:5|l0:\(int\)64, \(int\)1, \(bool\)0, \(int\)2, \(bool\)0:4}"
for spec in "${SPECS[@]}"; do
  name=${spec%%:*}; rest=${spec#*:}; rx=${rest%:*}; skip=${rest##*:}
  $NCU -k regex:"$rx" --launch-skip $skip -c 1 -o gpurun_out/prof_$name -f python tools/profile_sample.py 1024 > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
done

#!/bin/bash
# per-layer launch times (one forward, 1024 x 32) with and without MMAs, and a source-level
# ncu capture of the level-0 FiLM layer and a level-1 GN layer
cd "$(dirname "$0")/.."
O=gpurun_out/epi
mkdir -p $O
python tools/profile_unet.py 1024 1 > $O/plain.log 2>&1 || exit 1
for d in 0 2; do
  PS_TC_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,sm__cycles_active.avg --clock-control none --csv -k regex:unet_tc_kernel \
     --log-file $O/attr_$d.csv python tools/profile_unet.py 1024 1 > /dev/null 2>&1
  echo "dbg=$d rc=$?"
done
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:unet_tc_kernel --launch-skip 1 -c 1 -o $O/l0film -f python tools/profile_unet.py 1024 1 > $O/ncu_l0.log 2>&1; echo "l0 rc=$?"
$NCU -k regex:unet_tc_kernel --launch-skip 6 -c 1 -o $O/l1 -f python tools/profile_unet.py 1024 1 > $O/ncu_l1.log 2>&1; echo "l1 rc=$?"
for n in l0film l1; do
  ncu -i $O/$n.ncu-rep --page source --csv --print-source sass > $O/${n}_src.csv 2>/dev/null
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/${n}_raw.csv 2>/dev/null
done
ls -la $O

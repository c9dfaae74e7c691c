#!/bin/bash
# round-2 evidence: bench launch list, ncu --set full of the bench step's ESDF build + refinement
# and of one U-Net forward, strong-scaling proxies (per-rank problem counts on one GPU)
cd "$(dirname "$0")/.."
O=gpurun_out/r02
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > $O/bench_small.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_launch.log 2>&1
echo "launches rc=$?"
python tools/launch_summary.py $O/launches.csv $O/launches_summary.csv > /dev/null 2>&1; head -25 $O/launches_summary.csv
B1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"bl_refine|esdf_tile" -c 2 -o $O/prof_refine -f $B1 > $O/ncu_refine.log 2>&1
echo "refine ncu rc=$?"
python tools/refine_traffic.py $O/prof_refine.ncu-rep $O/refine_traffic.json
python tools/ncu_memory.py $O/prof_refine.ncu-rep $O/refine_esdf_ncu.csv > /dev/null 2>&1; cat $O/refine_esdf_ncu.csv
rm -f $O/prof_refine.ncu-rep
U="python tools/profile_unet.py 1024 1"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"unet_tc|xb_kernel|film_step" -c 31 -o $O/prof_unet -f $U > $O/ncu_unet.log 2>&1
echo "unet ncu rc=$?"
python tools/ncu_table.py $O/prof_unet.ncu-rep $O/unet_ncu_full.csv > /dev/null 2>&1
python tools/unet_traffic.py $O/prof_unet.ncu-rep $O/unet_traffic.json
rm -f $O/prof_unet.ncu-rep
for P in 128 256 512; do
  timeout 600 python bench.py --problems $P --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_p$P.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/bench_p$P.json')); print($P, round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
du -sh $O

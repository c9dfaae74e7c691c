#!/bin/bash
# final evidence of the round in one gpurun call (tests, smoke, bench repeats, launch list, ncu) (summaries only: ncu reports are reduced to CSV/JSON on the box)
cd "$(dirname "$0")/.."
O=gpurun_out/fin
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2>/dev/null; echo "reference rc=$?"
for i in 1 2 3 4 5; do
  timeout 600 python bench.py --steps 20 --warmup 5 $( [ $i = 1 ] || echo --no-cpu-baseline ) >> $O/bench_repeats.jsonl 2>/dev/null
done
python -c "import json; [print(round(json.loads(l)['value']), round(json.loads(l)['e2e']['value']), json.loads(l)['clocks']['sm_mhz']) for l in open('$O/bench_repeats.jsonl')]"
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_launch.log 2>&1
echo "launches rc=$?"
python tools/launch_summary.py $O/launches.csv $O/launches_summary.csv > /dev/null 2>&1; head -8 $O/launches_summary.csv
B1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"bl_refine|esdf_tile" -c 2 -o $O/prof_refine -f $B1 > $O/ncu_refine.log 2>&1
echo "refine ncu rc=$?"
python tools/refine_traffic.py $O/prof_refine.ncu-rep $O/refine_traffic.json
python tools/ncu_memory.py $O/prof_refine.ncu-rep $O/refine_esdf_ncu.csv > /dev/null 2>&1; cat $O/refine_esdf_ncu.csv
rm -f $O/prof_refine.ncu-rep
timeout 900 ncu --set full --clock-control none -k regex:"bl_refine" -c 4 -o $O/prof_cfg2 -f python tools/refine_cfg2_quad.py > $O/ncu_cfg2.log 2>&1
echo "cfg2 ncu rc=$?"
python tools/ncu_memory.py $O/prof_cfg2.ncu-rep $O/refine_cfg2_quad_ncu.csv > /dev/null 2>&1; cat $O/refine_cfg2_quad_ncu.csv
rm -f $O/prof_cfg2.ncu-rep
U="python tools/profile_unet.py 1024 1"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"unet_tc|xb_kernel" -c 31 -o $O/prof_unet -f $U > $O/ncu_unet.log 2>&1
echo "unet ncu rc=$?"
python tools/ncu_table.py $O/prof_unet.ncu-rep $O/unet_ncu_full.csv > /dev/null 2>&1
python tools/unet_traffic.py $O/prof_unet.ncu-rep $O/unet_traffic.json
rm -f $O/prof_unet.ncu-rep
for P in 128 256 512; do
  timeout 600 python bench.py --problems $P --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_p$P.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/bench_p$P.json')); print($P, round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
timeout 300 python tools/time_small_plan.py > $O/small_plan.json 2>&1; tail -3 $O/small_plan.json
du -sh $O

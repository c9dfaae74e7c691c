#!/bin/bash
# end-of-round evidence in one gpurun call (outputs kept small: ncu reports are summarised to
# CSV on the box and deleted -- gpurun copies back at most 64 MiB): GPU tests, bench line, bench
# launch list, ncu --set full of one U-Net forward and of the refinement / ESDF kernels,
# persistent-sampler trace, config-4 sweep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cat $O/bench.json
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > $O/bench_small.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_launch.log 2>&1
echo "launches rc=$?"
U="python tools/profile_unet.py 1024 1"
timeout 300 $U > $O/unet_plain.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"unet_tc|xb_kernel|film_step" -c 31 -o $O/prof_unet -f $U > $O/ncu_unet.log 2>&1
echo "unet ncu rc=$?"
python tools/ncu_table.py $O/prof_unet.ncu-rep $O/unet_ncu_full.csv > /dev/null 2>&1
python tools/unet_traffic.py $O/prof_unet.ncu-rep $O/unet_traffic.json > $O/unet_traffic.log 2>&1
ncu -i $O/prof_unet.ncu-rep --page details --csv > $O/unet_details.csv 2>/dev/null; gzip -f $O/unet_details.csv
rm -f $O/prof_unet.ncu-rep
R="python tools/time_refine.py"
timeout 300 $R > $O/refine_plain.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"bl_refine|esdf_cull" -c 6 -o $O/prof_refine -f $R > $O/ncu_refine.log 2>&1
echo "refine ncu rc=$?"
python tools/ncu_memory.py $O/prof_refine.ncu-rep $O/refine_esdf_ncu.csv
rm -f $O/prof_refine.ncu-rep
PS_NO_GRAPH=1 PS_PERSIST=1 PS_PERSIST_TRACE=$O/trace.bin timeout 300 python tools/persist_trace.py --run 1 32 && python tools/persist_trace.py $O/trace.bin 50 > $O/persist_trace.txt; echo "trace rc=$?"
rm -f $O/trace.bin
timeout 300 python tools/check_persist.py > $O/check_persist.log 2>&1; echo "check_persist rc=$?"
timeout 2400 python tools/sweep.py --out $O/sweep.json > $O/sweep.log 2>&1; echo "sweep rc=$?"
du -sh $O

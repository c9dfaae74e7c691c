cd /root/repo
NCU=0 bash tools/gpu_quick.sh
python tools/time_refine.py > gpurun_out/refine_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"esdf_cull" --launch-skip 4 --launch-count 1 -o gpurun_out/prof_esdf -f python tools/time_refine.py > gpurun_out/ncu_esdf.log 2>&1; echo esdf ncu rc=$?

cd /root/repo
U="python tools/profile_unet.py 1 3"
timeout 300 $U > gpurun_out/unet_plain_small.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fwd_launches_small.csv $U > /dev/null 2>&1; echo rc=$?
U="python tools/profile_unet.py 64 3"
timeout 300 $U > gpurun_out/unet_plain_small.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fwd_launches_c1.csv $U > /dev/null 2>&1; echo rc=$?

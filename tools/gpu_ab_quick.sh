#!/bin/bash
# U-Net change check: tc/sampler/planner tests on the working build, A/B of bench throughput
# against LIBS builds (name=path ...) at 1024 problems (and SMALL problems if set), one-forward
# per-layer launch times of the working build
cd "$(dirname "$0")/.."
O=gpurun_out/ab
mkdir -p $O
timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_sampler_gpu.py tests/test_planner_gpu.py ${EXTRA_TESTS} -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
ROUNDS=${ROUNDS:-3} LIBS="$LIBS" BENCH_ARGS="--steps 10 --warmup 3" bash tools/ab_multi.sh 2>&1 | tee $O/ab.txt
if [ -n "$SMALL" ]; then
  echo "--- problems $SMALL"
  ROUNDS=${ROUNDS:-3} LIBS="$LIBS" BENCH_ARGS="--steps 10 --warmup 3 --problems $SMALL" bash tools/ab_multi.sh 2>&1 | tee $O/ab_small.txt
fi
if [ "${ATTR:-1}" = 1 ]; then
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum --clock-control none --csv -k regex:unet_tc_kernel \
   --log-file $O/attr.csv python tools/profile_unet.py 1024 1 > /dev/null 2>&1; echo "attr rc=$?"
python tools/attr_table.py $O/attr.csv | tail -1
fi

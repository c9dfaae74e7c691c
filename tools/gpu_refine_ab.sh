#!/bin/bash
# refinement change check: bl tests on the working build, refine timings of LIBS builds vs head
cd "$(dirname "$0")/.."
O=gpurun_out/rab
mkdir -p $O
timeout 900 python -m pytest tests/test_bl_gpu.py tests/test_guided_gpu.py tests/test_planner_gpu.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for i in 1 2; do
for spec in head ${LIBS}; do
  name=${spec%%=*}; path=${spec#*=}
  if [ $name = head ]; then unset PS_LIB_OVERRIDE; else export PS_LIB_OVERRIDE=$PWD/$path; fi
  echo "$name $(timeout 600 python tools/time_refine.py 2>/dev/null | tail -1)"
done
done

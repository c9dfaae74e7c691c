#!/bin/bash
# A/B: the working build vs LIBS builds, and the working build with KNOB set (ROUNDS alternations)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_sampler_gpu.py -x -q > gpurun_out/ab/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ab/pytest.log
if [ -n "$KNOB" ]; then env $KNOB timeout 900 python -m pytest tests/test_tc_gpu.py -x -q > gpurun_out/ab/pytest_knob.log 2>&1; echo "pytest knob rc=$?"; tail -1 gpurun_out/ab/pytest_knob.log; fi
for i in $(seq ${ROUNDS:-3}); do
  for spec in head ${LIBS} ${KNOB:+knob}; do
    name=${spec%%=*}; path=${spec#*=}
    unset PS_LIB_OVERRIDE
    if [ $name = knob ]; then E="$KNOB"; elif [ $name = head ]; then E=""; else E="PS_LIB_OVERRIDE=$PWD/$path"; fi
    env $E python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value']), round(d['roofline']['sampler_ms'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])"
  done
done

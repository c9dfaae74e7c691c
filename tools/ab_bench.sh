#!/bin/bash
# A/B device throughput of the working build vs abtmp/libps_prev.so (same box, alternating)
cd "$(dirname "$0")/.."
for i in $(seq ${ROUNDS:-2}); do
  for v in new prev; do
    if [ $v = prev ]; then export PS_LIB_OVERRIDE=$PWD/abtmp/libps_prev.so; else unset PS_LIB_OVERRIDE; fi
    python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['roofline']['sampler_ms'],1), d['ms_per_step'], d['clocks']['sm_mhz'])"
  done
done

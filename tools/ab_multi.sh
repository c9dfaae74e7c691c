#!/bin/bash
# device throughput of several builds on one box: LIBS="name=path ..." (the working build is "head")
cd "$(dirname "$0")/.."
for i in $(seq ${ROUNDS:-1}); do
  for spec in head ${LIBS}; do
    name=${spec%%=*}; path=${spec#*=}
    if [ $name = head ]; then unset PS_LIB_OVERRIDE; else export PS_LIB_OVERRIDE=$PWD/$path; fi
    python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value']), round(d['roofline']['sampler_ms'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])"
  done
done

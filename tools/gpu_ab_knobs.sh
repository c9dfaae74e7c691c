#!/bin/bash
# A/B of env knobs on the working build: KNOBS="A=1 A=3 ..." (each a single NAME=VALUE), ROUNDS alternations
cd "$(dirname "$0")/.."
for k in $KNOBS; do
  env $k timeout 900 python -m pytest tests/test_tc_gpu.py -x -q > /tmp/pt.log 2>&1; echo "pytest $k rc=$? $(tail -1 /tmp/pt.log)"
done
for i in $(seq ${ROUNDS:-3}); do
  for k in default $KNOBS; do
    E=""; [ $k != default ] && E=$k
    env $E python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', round(d['value']), round(d['roofline']['sampler_ms'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])"
  done
done

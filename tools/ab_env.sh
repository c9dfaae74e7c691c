#!/bin/bash
# A/B device throughput: default vs an env knob (KNOB="NAME=1"), same box, alternating
cd "$(dirname "$0")/.."
for i in $(seq ${ROUNDS:-2}); do
  python bench.py --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', round(d['value']), round(d['e2e']['value']), round(d['roofline']['sampler_ms'],1), d['clocks']['sm_mhz'])"
  env $KNOB python bench.py --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$KNOB', round(d['value']), round(d['e2e']['value']), round(d['roofline']['sampler_ms'],1), d['clocks']['sm_mhz'])"
done

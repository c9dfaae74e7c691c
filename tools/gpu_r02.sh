#!/bin/bash
# round-2 GPU check: full -m gpu suite, agreement rates, one bench run (each bounded by timeout)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q -rA ${PYTEST_ARGS} --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log | grep -v "^PASSED"
if [ -n "${AGREE}" ]; then
timeout 900 python tools/agreement.py ${AGREE} > gpurun_out/agreement.json 2> gpurun_out/agreement.err; echo "agreement rc=$?"; cat gpurun_out/agreement.json; tail -3 gpurun_out/agreement.err
fi
if [ "${BENCH:-1}" = 1 ]; then
timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
fi

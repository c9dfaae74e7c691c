# per-layer critical path of the persistent sampler under PS_TC_DBG knobs (1 no epilogue, 2 no MMA, 16 no weight loads)
cd /root/repo
for d in ${DBGS:-0 2 16 1}; do
  echo "== PS_TC_DBG=$d"
  PS_TC_DBG=$d PS_NO_GRAPH=1 PS_PERSIST=1 PS_PERSIST_TRACE=gpurun_out/trace_$d.bin timeout 300 python tools/persist_trace.py --run ${P:-1} ${S:-32} && python tools/persist_trace.py gpurun_out/trace_$d.bin 50
done

cd /root/repo
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
PS_NO_GRAPH=1 PS_PERSIST=1 PS_PERSIST_TRACE=gpurun_out/trace_n.bin timeout 300 python tools/persist_trace.py --run 1 32 && python tools/persist_trace.py gpurun_out/trace_n.bin 50 | grep -E "^ +(0|1|6|11|12|18|27|28) |step total"
timeout 300 python tools/check_persist.py 2>&1 | grep time | head -4
timeout 300 python tools/time_refine.py
PS_REFINE_THREADS=128 timeout 300 python tools/time_refine.py
timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value']), round(d['e2e']['value']), round(d['roofline']['sampler_ms'],1), d['ms_per_step'], d['clocks'])"
rm -f gpurun_out/trace_n.bin

timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "attention" 2>&1 | tail -1
ELIS_LIB=libelis_atrace.so timeout 300 python scripts/attn64_trace.py 1311 2>&1
for rep in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('cfg5', d['ms_per_step'], 'attn', round(k['attention'],3), 'clk', d['clocks']['sm_mhz'])"
done

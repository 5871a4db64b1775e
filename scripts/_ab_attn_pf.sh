# attention (64-key engine): L2 prefetch of the later key blocks at CTA start (default) vs none
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "attention" 2>&1 | tail -1
for rep in 1 2; do
for v in default nopf; do
  lib=libelis_$v.so; [ $v = default ] && lib=libelis.so
  ELIS_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$v cfg5', d['ms_per_step'], 'attn', round(k['attention'],3), 'clk', d['clocks']['sm_mhz'])"
  ELIS_LIB=$lib timeout 200 python bench.py --workload cfg2 --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$v cfg2', d['ms_per_step'], 'attn', round(k['attention'],3), 'clk', d['clocks']['sm_mhz'])"
done
done

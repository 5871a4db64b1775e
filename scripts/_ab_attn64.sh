# attention: 64-key-block engine (O in TMEM, default) vs the round-1 128-key-block engine (ELIS_ATTN_ENGINE=128)
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "attention" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_predict.py tests/test_gpu_residual16.py tests/test_gpu_fp8.py tests/test_gpu_cls_prune.py -q -x 2>&1 | grep -E "^E |passed|failed" | head -5
for rep in 1 2; do
for e in 64 128; do
  ELIS_ATTN_ENGINE=$e timeout 200 python bench.py --workload cfg2 --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('engine $e cfg2', d['ms_per_step'], 'attn', round(k['attention'],3), 'clk', d['clocks']['sm_mhz'])"
done
done
for e in 64 128; do
  ELIS_ATTN_ENGINE=$e timeout 300 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('engine $e cfg5', d['ms_per_step'], 'attn', round(k['attention'],3), 'clk', d['clocks']['sm_mhz'])"
done

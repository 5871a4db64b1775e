# A/B: packed fp32x2 LN / bias / residual epilogue math (default) vs scalar (libelis_gx2: packed GELU only)
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_residual16.py -q -x 2>&1 | tail -1
for rep in 1 2; do
for v in default gx2; do
  lib=libelis_$v.so; [ $v = default ] && lib=libelis.so
  ELIS_LIB=$lib timeout 200 python bench.py --workload cfg2 --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$v cfg2', d['ms_per_step'], 'ffn1', round(k['gemm_ffn1'],3), 'ffn2', round(k['gemm_ffn2'],3), 'out', round(k['gemm_out'],3), 'qkv', round(k['gemm_qkv'],3), 'clk', d['clocks']['sm_mhz'])"
done
done
for v in default gx2; do
  lib=libelis_$v.so; [ $v = default ] && lib=libelis.so
  ELIS_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$v cfg5', d['ms_per_step'], 'ffn1', round(k['gemm_ffn1'],3), 'ffn2', round(k['gemm_ffn2'],3), 'out', round(k['gemm_out'],3), 'qkv', round(k['gemm_qkv'],3), 'clk', d['clocks']['sm_mhz'])"
done

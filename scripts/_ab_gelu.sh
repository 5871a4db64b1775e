# A/B: FFN1 GELU epilogue -- scalar sigmoid form (default), packed fp32x2 sigmoid form, tanh form (1 MUFU)
for rep in 1 2; do
for v in default gx2 gtanh; do
  lib=libelis_$v.so; [ $v = default ] && lib=libelis.so
  ELIS_LIB=$lib timeout 200 python bench.py --workload cfg2 --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$v cfg2', d['ms_per_step'], 'ffn1', round(k['gemm_ffn1'],3), 'qkv', round(k['gemm_qkv'],3), 'clk', d['clocks']['sm_mhz'])"
done
done
ELIS_LIB=libelis_gx2.so timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "gemm and (1 or epi)" 2>&1 | tail -1
ELIS_LIB=libelis_gtanh.so timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "gemm_f16" 2>&1 | tail -1

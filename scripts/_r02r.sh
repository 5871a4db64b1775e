timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_residual16.py tests/test_gpu_fp16.py tests/test_gpu_predict.py tests/test_gpu_fp8.py tests/test_gpu_cls_prune.py -q -x 2>&1 | grep -E "^E |FAILED|passed|failed" | head
for v in default gx2; do
  lib=libelis_$v.so; [ $v = default ] && lib=libelis.so
  ELIS_LIB=$lib timeout 200 python bench.py --workload cfg2 --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$v cfg2', d['ms_per_step'], 'ffn1', round(k['gemm_ffn1'],3), 'ffn2', round(k['gemm_ffn2'],3), 'out', round(k['gemm_out'],3), 'clk', d['clocks']['sm_mhz'])"
done

# A/B: LN statistics exchange with st.async + transaction barrier (default build) vs release arrives
set -x
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fp8.py -q -x -k "layernorm or ln" 2>&1 | tail -2
for i in 1 2; do
  for lib in libelis.so libelis_relarr.so; do
    ELIS_LIB=$lib timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_step']; print('$lib', d['ms_per_step'], 'out', k['gemm_out'], 'ffn2', k['gemm_ffn2'])"
  done
done
ELIS_LIB=libelis_gtrace.so timeout 300 python scripts/gemm_trace.py --r16 2>&1 | tail -6

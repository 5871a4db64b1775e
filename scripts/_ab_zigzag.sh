# A/B: QKV / FFN1 M tiles in descending order (default; ELIS_GEMM_ZIGZAG=0 ascending): first read the A rows the producer wrote last
ELIS_GEMM_ZIGZAG=1 timeout 600 python -m pytest tests/test_gpu_predict.py tests/test_gpu_residual16.py -q -x -k "ragged or invariance or cfg2 or residual16_base" 2>&1 | tail -1
for i in 1 2 3; do
  for z in 0 1; do
    ELIS_GEMM_ZIGZAG=$z timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_step']; print('zigzag=$z', d['ms_per_step'], 'qkv', k['gemm_qkv'], 'ffn1', k['gemm_ffn1'], 'ffn2', k['gemm_ffn2'], 'pass', d['kernels_pass_ms_per_step'])"
  done
done

# A/B: FFN2 LN statistics through global memory on 144 SMs (ELIS_GEMM_GX=1) vs the 6-CTA cluster exchange (default)
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "global_stats or residual16" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_residual16.py tests/test_gpu_predict.py -q -x -k "residual16 or r16" 2>&1 | tail -2
for i in 1 2; do
  for gx in 1 0; do
    ELIS_GEMM_GX=$gx timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_step']; print('gx=$gx', d['ms_per_step'], 'out', k['gemm_out'], 'ffn2', k['gemm_ffn2'])"
  done
done

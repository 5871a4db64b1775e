# round-2l: new per-op fp16 GEMM tests, cfg2 hidden states on 32 requests, compute-sanitizer runs
set -x
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "gemm_f16" > gpurun_out/r02l_gemm_f16.log 2>&1; tail -2 gpurun_out/r02l_gemm_f16.log
timeout 900 python -m pytest tests/test_gpu_predict.py -q -s -k "hidden_states_32" > gpurun_out/r02l_hidden32.log 2>&1; grep -E "hidden max|passed|failed" gpurun_out/r02l_hidden32.log
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_run.py > gpurun_out/r02l_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r02l_sanitizer_$tool.log
done

# optional attention engines bitwise vs default; compute-sanitizer on the final build
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention_engines.py -q 2>&1 | tail -2 | tee gpurun_out/r02zl_engines_test.txt
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_run.py > gpurun_out/r02zl_sanitizer_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error' gpurun_out/r02zl_sanitizer_$tool.log | tail -2)"
done

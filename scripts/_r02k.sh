set -x
timeout 600 python -m pytest tests/test_gpu_predict.py tests/test_gpu_residual16.py tests/test_gpu_fp16.py -x -q > gpurun_out/r02k_tests.log 2>&1; tail -1 gpurun_out/r02k_tests.log
for a in "--workload cfg2" ""; do
timeout 200 python bench.py $a --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$a', d['ms_per_step'], 'embed', round(d['kernels_ms_per_step']['embed_ln'],3))"
done

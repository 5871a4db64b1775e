set -x
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_predict.py -x -q -k "fc or predict" > gpurun_out/r02j_tests.log 2>&1; tail -1 gpurun_out/r02j_tests.log
for a in "--workload cfg2" "" "--requests 164"; do
timeout 200 python bench.py $a --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$a', d['ms_per_step'], 'head_fc', round(d['kernels_ms_per_step']['head_fc'],3))"
done

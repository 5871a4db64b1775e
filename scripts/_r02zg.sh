# pool unroll (default lib) + head FC ring depth A/B (ELIS_HEAD_STAGES 2 / 3 / 4)
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_predict.py -q -x -k "pool or fc or head or predict" 2>&1 | tail -2
for lib in libelis.so libelis_hs3.so libelis_hs4.so; do
  ELIS_LIB=$lib timeout 200 python scripts/small_predict_latency.py --ns 4,64,1311 --iters 100 | sed "s/^/$lib /"
  ELIS_LIB=$lib timeout 150 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$lib cfg5', d['ms_per_step'], 'head_fc', round(k['head_fc'],4), 'pool', round(k['pool'],4), 'clk', d['clocks']['sm_mhz'])"
done 2>&1 | tee gpurun_out/r02zg_head_stages.txt

# FFN1 GELU: packed tanh form (1 MUFU per element, default) vs the packed sigmoid form (libelis_gs.so)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_predict.py tests/test_gpu_residual16.py tests/test_gpu_fp16.py -q -x 2>&1 | tail -2
for rep in 1 2 3; do
for lib in libelis_gs.so libelis.so; do
  ELIS_LIB=$lib timeout 150 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$lib cfg5', d['ms_per_step'], 'ffn1', round(k['gemm_ffn1'],3), 'clk', d['clocks']['sm_mhz'])"
  ELIS_LIB=$lib timeout 100 python bench.py --workload cfg2 --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$lib cfg2', d['ms_per_step'], 'ffn1', round(k['gemm_ffn1'],3), 'clk', d['clocks']['sm_mhz'])"
done
done 2>&1 | tee gpurun_out/r02zm_ab_gelu_tanh2.txt
timeout 1200 python scripts/parity_sweep.py --seeds 10 --paths fp16-r16 > gpurun_out/r02zm_parity_sweep.jsonl 2>&1; tail -3 gpurun_out/r02zm_parity_sweep.jsonl

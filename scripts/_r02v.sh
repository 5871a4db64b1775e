# PDL A/B (ELIS_PDL=0 vs default on) + tcgen05 SS/TS MMA rate microbenchmark
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2505_09142_b200/csrc scripts/tc_rate.cu -o /tmp/tc_rate && timeout 60 /tmp/tc_rate > gpurun_out/r02v_tc_rate.txt 2>&1
cat gpurun_out/r02v_tc_rate.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_graph.py tests/test_gpu_predict.py tests/test_gpu_residual16.py -q -x 2>&1 | tail -2
for rep in 1 2; do
for p in 0 1; do
  ELIS_PDL=$p timeout 300 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('pdl $p cfg5', d['ms_per_step'], 'attn', round(k['attention'],3), 'clk', d['clocks']['sm_mhz'])"
  ELIS_PDL=$p timeout 200 python bench.py --workload cfg2 --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pdl $p cfg2', d['ms_per_step'], 'clk', d['clocks']['sm_mhz'])"
done
done 2>&1 | tee gpurun_out/r02v_ab_pdl.txt

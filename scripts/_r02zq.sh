# FFN2 LN statistics through global memory on all SMs (ELIS_GEMM_GX=1) at cfg5
for rep in 1 2 3; do
for gx in 0 1; do
  ELIS_GEMM_GX=$gx timeout 150 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('gx $gx cfg5', d['ms_per_step'], 'ffn2', round(k['gemm_ffn2'],3), 'clk', d['clocks']['sm_mhz'])"
done
done 2>&1 | tee gpurun_out/r02zq_ab_gx_ffn2_cfg5.txt

# exp2 split retune after the warp-elect MMA issue: pairs of 16 on the FMA pipe = 2 / 4 / 6 (default) / 8
for rep in 1 2; do
for lib in libelis_p2.so libelis_p4.so libelis.so libelis_p8.so; do
  ELIS_LIB=$lib timeout 150 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$lib cfg5', d['ms_per_step'], 'attn', round(k['attention'],3), 'clk', d['clocks']['sm_mhz'])"
  ELIS_LIB=$lib timeout 100 python bench.py --workload cfg2 --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$lib cfg2', d['ms_per_step'], 'attn', round(k['attention'],3), 'clk', d['clocks']['sm_mhz'])"
done
done 2>&1 | tee gpurun_out/r02zo_ab_exp2_split.txt

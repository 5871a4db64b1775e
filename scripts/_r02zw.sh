# embedding occupancy: __launch_bounds__(256, 5) (48 registers) vs the default (57)
for rep in 1 2; do
for lib in libelis.so libelis_e5.so; do
  ELIS_LIB=$lib timeout 150 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$lib cfg5', d['ms_per_step'], 'embed', round(k['embed_ln'],4), 'clk', d['clocks']['sm_mhz'])"
done
done 2>&1 | tee gpurun_out/r02zw_embed_occupancy.txt
for lib in libelis.so libelis_e5.so; do ELIS_LIB=$lib timeout 90 python scripts/run_predict.py --n 256 --iters 1 --dump /tmp/c2_$lib.npz | tail -1; done
python -c "
import numpy as np
a,b=np.load('/tmp/c2_libelis.so.npz'),np.load('/tmp/c2_libelis_e5.so.npz')
print('bitwise', np.array_equal(a['pred'].view(np.uint32),b['pred'].view(np.uint32)), np.array_equal(a['hidden'].view(np.uint32),b['hidden'].view(np.uint32)))" | tee -a gpurun_out/r02zw_embed_occupancy.txt

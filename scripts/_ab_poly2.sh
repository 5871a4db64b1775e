# A/B: share of exp2 pairs on the FMA pipe in the persistent attention engine (0, 3, 6 of 16)
for rep in 1 2; do
for v in p0 p3 default; do
  lib=libelis_$v.so; [ $v = default ] && lib=libelis.so
  ELIS_LIB=$lib timeout 200 python bench.py --workload cfg2 --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v cfg2', d['ms_per_step'], 'attn', round(d['kernels_ms_per_step']['attention'],3))"
done
done

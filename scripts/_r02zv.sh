# PDL on pool and head_out: full GPU suite + small-predict latency (PDL on / off)
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
for p in 0 1; do ELIS_PDL=$p timeout 200 python scripts/small_predict_latency.py --ns 1,4,64 --iters 100 | sed "s/^/pdl=$p /"; done 2>&1 | tee gpurun_out/r02zv_pool_headout_pdl.txt
timeout 100 python bench.py --workload cfg1 --no-cpu-baseline --steps 50 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg1', d['ms_per_step'])" | tee -a gpurun_out/r02zv_pool_headout_pdl.txt

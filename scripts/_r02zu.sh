# PDL on the 3xTF32 head FC chain
for p in 0 1 0 1; do ELIS_PDL=$p timeout 200 python scripts/small_predict_latency.py --ns 1,4,64 --iters 100 | sed "s/^/pdl=$p /"; done 2>&1 | tee gpurun_out/r02zu_head_pdl.txt
for p in 0 1; do ELIS_PDL=$p timeout 100 python bench.py --workload cfg1 --no-cpu-baseline --steps 50 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pdl $p cfg1', d['ms_per_step'])"; done 2>&1 | tee -a gpurun_out/r02zu_head_pdl.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_predict.py tests/test_gpu_graph.py -q -x -k "fc or head or predict or graph or invarian" 2>&1 | tail -2

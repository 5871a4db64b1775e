set -x
timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_scheduler.py tests/test_gpu_streamsim.py tests/test_gpu_table.py tests/test_gpu_peer.py tests/test_gpu_dist.py -q -x 2>&1 | tail -3
timeout 1200 python scripts/short_request_parity.py > gpurun_out/r02n_short_parity.jsonl 2> gpurun_out/r02n_short_parity.err; cat gpurun_out/r02n_short_parity.jsonl; tail -3 gpurun_out/r02n_short_parity.err
timeout 200 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg5', d['ms_per_step'], {k: round(v,3) for k,v in d['kernels_ms_per_step'].items() if 'select' in k or 'head' in k})"

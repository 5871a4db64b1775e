# round-2g: decoupled S / P attention pipeline: parity first (bounded), then trace + bench
set -x
timeout 120 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" > gpurun_out/r02g_tests.log 2>&1; rc=$?; tail -2 gpurun_out/r02g_tests.log
if [ $rc -ne 0 ]; then grep -E "Error|assert" gpurun_out/r02g_tests.log | head; exit 1; fi
ELIS_LIB=libelis_atrace.so timeout 60 python scripts/attn_trace.py 256 > gpurun_out/r02g_trace.txt 2>&1
timeout 200 python bench.py --workload cfg2 --no-cpu-baseline --steps 10 > gpurun_out/r02g_bench_cfg2.json 2> gpurun_out/r02g_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02g_bench_cfg2.json").read().strip().splitlines()[-1])
print("cfg2", d["ms_per_step"], {k: round(v, 3) for k, v in d["kernels_ms_per_step"].items()})
PY
cat gpurun_out/r02g_trace.txt

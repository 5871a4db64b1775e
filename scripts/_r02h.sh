# round-2h: 3xTF32 tensor-core head: parity, then bench cfg2 / cfg5
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02h_gpu_tests.log 2>&1; rc=$?; tail -3 gpurun_out/r02h_gpu_tests.log
if [ $rc -ne 0 ]; then grep -E "Error|assert|FAILED" gpurun_out/r02h_gpu_tests.log | head -20; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; tail -1 gpurun_out/r02h_smoke.log
timeout 200 python bench.py --workload cfg2 --no-cpu-baseline --steps 10 > gpurun_out/r02h_bench_cfg2.json 2> gpurun_out/r02h_bench.err
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/r02h_bench_cfg5.json 2>> gpurun_out/r02h_bench.err
timeout 200 python bench.py --no-cpu-baseline --steps 10 --requests 164 > gpurun_out/r02h_bench_cfg5_due164.json 2>> gpurun_out/r02h_bench.err
python - <<'PY'
import json
for f in ("cfg2", "cfg5", "cfg5_due164"):
    try:
        d = json.loads(open(f"gpurun_out/r02h_bench_{f}.json").read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], {k: round(v, 3) for k, v in d["kernels_ms_per_step"].items()})
    except Exception as e:
        print(f, "failed", e)
PY

# round-2c: persistent two-pipeline attention with packed short requests -- parity + bench
set -x
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" > gpurun_out/r02c_attn_tests.log 2>&1; tail -5 gpurun_out/r02c_attn_tests.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02c_gpu_tests.log 2>&1; tail -5 gpurun_out/r02c_gpu_tests.log
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/r02c_bench_cfg2.json 2> gpurun_out/r02c_bench.err
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02c_bench_cfg5.json 2>> gpurun_out/r02c_bench.err
tail -3 gpurun_out/r02c_bench.err
python - <<'PY'
import json
for f in ("cfg2", "cfg5"):
    try:
        d = json.loads(open(f"gpurun_out/r02c_bench_{f}.json").read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], {k: round(v, 3) for k, v in d["kernels_ms_per_step"].items()})
    except Exception as e:
        print(f, "failed", e)
PY

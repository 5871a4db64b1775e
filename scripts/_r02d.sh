# round-2d: attention grid = one CTA per SM; parity, bench, ncu of one attention launch
set -x
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_predict.py -x -q > gpurun_out/r02d_tests.log 2>&1; tail -3 gpurun_out/r02d_tests.log
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/r02d_bench_cfg2.json 2> gpurun_out/r02d_bench.err
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02d_bench_cfg5.json 2>> gpurun_out/r02d_bench.err
python - <<'PY'
import json
for f in ("cfg2", "cfg5"):
    try:
        d = json.loads(open(f"gpurun_out/r02d_bench_{f}.json").read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], {k: round(v, 3) for k, v in d["kernels_ms_per_step"].items()})
    except Exception as e:
        print(f, "failed", e)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_attention_tc" -s 2 -c 1 \
  -o gpurun_out/r02d_attn -f python scripts/run_predict.py --iters 1 > gpurun_out/r02d_ncu.log 2>&1
tail -2 gpurun_out/r02d_ncu.log

# early-S attention engine (ELIS_ATTN_ENGINE=66, default) vs the 64-key engine (64): hang check,
# tests, bitwise equality, A/B timing
mkdir -p gpurun_out
for L in 1 "1,2" "130" "1,2,63,64,65,130,7,512,200,33" "512,511,257,100,3" trace:1311; do
  timeout 30 python scripts/attn_repro.py $L 2>&1 | grep -v Warn | tail -2 | tee /tmp/rep.txt
  grep -q "^ok" /tmp/rep.txt || { echo "attention repro failed for $L"; exit 1; }
done
timeout 120 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -3
for e in 64 66; do
  ELIS_ATTN_ENGINE=$e timeout 90 python scripts/run_predict.py --n 256 --iters 1 --dump /tmp/cfg2_$e.npz | tail -1
  ELIS_ATTN_ENGINE=$e timeout 90 python scripts/run_predict.py --workload cfg5 --iters 1 --dump /tmp/cfg5_$e.npz | tail -1
  ELIS_ATTN_ENGINE=$e timeout 90 python scripts/run_predict.py --n 512 --lengths uniform --precision bf16 --iters 1 --dump /tmp/bf_$e.npz | tail -1
done
python - <<'PY' 2>&1 | tee gpurun_out/r02z_attn_engine_bitwise.txt
import numpy as np
for w in ("cfg2", "cfg5", "bf"):
    a, b = np.load(f"/tmp/{w}_64.npz"), np.load(f"/tmp/{w}_66.npz")
    print(w, "pred bitwise equal:", np.array_equal(a["pred"].view(np.uint32), b["pred"].view(np.uint32)),
          "hidden bitwise equal:", np.array_equal(a["hidden"].view(np.uint32), b["hidden"].view(np.uint32)))
PY
for rep in 1 2; do
for e in 64 66; do
  ELIS_ATTN_ENGINE=$e timeout 150 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('engine $e cfg5', d['ms_per_step'], 'attn', round(k['attention'],3), 'clk', d['clocks']['sm_mhz'])"
  ELIS_ATTN_ENGINE=$e timeout 100 python bench.py --workload cfg2 --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('engine $e cfg2', d['ms_per_step'], 'attn', round(k['attention'],3), 'clk', d['clocks']['sm_mhz'])"
done
done 2>&1 | tee gpurun_out/r02z_ab_attn_early_s.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_predict.py tests/test_gpu_residual16.py tests/test_gpu_fp8.py tests/test_gpu_graph.py tests/test_gpu_cls_prune.py -q -x 2>&1 | tail -3

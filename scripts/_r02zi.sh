# embedding over the work-list tiles (default) vs per-token search (ELIS_EMBED_TILES=0)
mkdir -p gpurun_out
for e in 0 1; do
  ELIS_EMBED_TILES=$e timeout 90 python scripts/run_predict.py --n 256 --iters 1 --dump /tmp/cfg2_e$e.npz | tail -1
  ELIS_EMBED_TILES=$e timeout 90 python scripts/run_predict.py --workload cfg5 --iters 1 --dump /tmp/cfg5_e$e.npz | tail -1
  ELIS_EMBED_TILES=$e timeout 90 python scripts/run_predict.py --config tiny --n 16 --lengths fixed:64 --iters 1 --dump /tmp/tiny_e$e.npz | tail -1
  ELIS_EMBED_TILES=$e timeout 90 python scripts/run_predict.py --config large --n 64 --lengths uniform --iters 1 --dump /tmp/large_e$e.npz | tail -1
done
python - <<'PY' 2>&1 | tee gpurun_out/r02zi_embed_tiles_bitwise.txt
import numpy as np
for w in ("cfg2", "cfg5", "tiny", "large"):
    a, b = np.load(f"/tmp/{w}_e0.npz"), np.load(f"/tmp/{w}_e1.npz")
    print(w, "pred bitwise equal:", np.array_equal(a["pred"].view(np.uint32), b["pred"].view(np.uint32)),
          "hidden bitwise equal:", np.array_equal(a["hidden"].view(np.uint32), b["hidden"].view(np.uint32)))
PY
for rep in 1 2; do
for e in 0 1; do
  ELIS_EMBED_TILES=$e timeout 150 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('embed_tiles $e cfg5', d['ms_per_step'], 'embed', round(k['embed_ln'],4), 'clk', d['clocks']['sm_mhz'])"
done
done 2>&1 | tee gpurun_out/r02zi_ab_embed_tiles.txt
ELIS_EMBED_TILES=1 timeout 200 python scripts/small_predict_latency.py --ns 4,64 --iters 100
timeout 900 python -m pytest tests/test_gpu_predict.py tests/test_gpu_residual16.py tests/test_gpu_fp8.py tests/test_gpu_graph.py tests/test_gpu_cls_prune.py tests/test_gpu_fp16.py tests/test_gpu_arena.py -q -x 2>&1 | tail -2

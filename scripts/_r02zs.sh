# small-M 256 x 128 tiles for QKV / FFN1 (default) vs 256 x 256 (ELIS_GEMM_SMALLM=0): bitwise + latency
mkdir -p gpurun_out
for sm in 0 1; do
  for n in 4 16 64; do
    ELIS_GEMM_SMALLM=$sm timeout 90 python scripts/run_predict.py --n $n --iters 1 --dump /tmp/n${n}_sm$sm.npz | tail -1
  done
done
python - <<'PY' 2>&1 | tee gpurun_out/r02zs_smallm_bitwise.txt
import numpy as np
for n in (4, 16, 64):
    a, b = np.load(f"/tmp/n{n}_sm0.npz"), np.load(f"/tmp/n{n}_sm1.npz")
    print(n, "requests: 256x128 vs 256x256 tiles: pred bitwise equal:", np.array_equal(a["pred"].view(np.uint32), b["pred"].view(np.uint32)),
          "hidden bitwise equal:", np.array_equal(a["hidden"].view(np.uint32), b["hidden"].view(np.uint32)))
PY
for sm in 0 1 0 1; do ELIS_GEMM_SMALLM=$sm timeout 200 python scripts/small_predict_latency.py --ns 1,4,16,64 --iters 100 | sed "s/^/smallm=$sm /"; done 2>&1 | tee gpurun_out/r02zs_small_predict.txt
timeout 900 python -m pytest tests/test_gpu_predict.py tests/test_gpu_residual16.py tests/test_gpu_graph.py tests/test_gpu_fp16.py tests/test_gpu_streamsim.py -q -x 2>&1 | tail -2

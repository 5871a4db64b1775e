# out-projection LN statistics through global memory on every SM (ELIS_GEMM_GX_OUT=1) vs the
# 132-SM cluster exchange: bitwise check + A/B
mkdir -p gpurun_out
for gx in 0 1; do
  ELIS_GEMM_GX_OUT=$gx timeout 90 python scripts/run_predict.py --n 256 --iters 1 --dump /tmp/cfg2_gx$gx.npz | tail -1
  ELIS_GEMM_GX_OUT=$gx timeout 90 python scripts/run_predict.py --workload cfg5 --iters 1 --dump /tmp/cfg5_gx$gx.npz | tail -1
done
python - <<'PY' 2>&1 | tee gpurun_out/r02zh_gx_out_bitwise.txt
import numpy as np
for w in ("cfg2", "cfg5"):
    a, b = np.load(f"/tmp/{w}_gx0.npz"), np.load(f"/tmp/{w}_gx1.npz")
    print(w, "pred bitwise equal:", np.array_equal(a["pred"].view(np.uint32), b["pred"].view(np.uint32)),
          "hidden bitwise equal:", np.array_equal(a["hidden"].view(np.uint32), b["hidden"].view(np.uint32)))
PY
for rep in 1 2 3; do
for gx in 0 1; do
  ELIS_GEMM_GX_OUT=$gx timeout 150 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('gx_out $gx cfg5', d['ms_per_step'], 'out', round(k['gemm_out'],3), 'clk', d['clocks']['sm_mhz'])"
  ELIS_GEMM_GX_OUT=$gx timeout 100 python bench.py --workload cfg2 --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('gx_out $gx cfg2', d['ms_per_step'], 'out', round(k['gemm_out'],3), 'clk', d['clocks']['sm_mhz'])"
done
done 2>&1 | tee gpurun_out/r02zh_ab_gx_out.txt

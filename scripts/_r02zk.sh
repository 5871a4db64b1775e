# attention MMA issue: warp 0 converged + elect (default) vs thread 0 (libelis_wi0.so)
mkdir -p gpurun_out
for L in 1 "1,2,63,64,65,130,7,512,200,33" trace:1311; do
  timeout 30 python scripts/attn_repro.py $L 2>&1 | grep -v Warn | tail -1 | cut -c1-50 | tee /tmp/rep.txt
  grep -q "^ok" /tmp/rep.txt || { echo "attention repro failed for $L"; exit 1; }
done
timeout 120 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -1
for lib in libelis_wi0.so libelis.so; do
  ELIS_LIB=$lib timeout 90 python scripts/run_predict.py --n 256 --iters 1 --dump /tmp/cfg2_$lib.npz | tail -1
  ELIS_LIB=$lib timeout 90 python scripts/run_predict.py --workload cfg5 --iters 1 --dump /tmp/cfg5_$lib.npz | tail -1
done
python - <<'PY' 2>&1 | tee gpurun_out/r02zk_warp_issue_bitwise.txt
import numpy as np
for w in ("cfg2", "cfg5"):
    a, b = np.load(f"/tmp/{w}_libelis_wi0.so.npz"), np.load(f"/tmp/{w}_libelis.so.npz")
    print(w, "pred bitwise equal:", np.array_equal(a["pred"].view(np.uint32), b["pred"].view(np.uint32)),
          "hidden bitwise equal:", np.array_equal(a["hidden"].view(np.uint32), b["hidden"].view(np.uint32)))
PY
for rep in 1 2 3; do
for lib in libelis_wi0.so libelis.so; do
  ELIS_LIB=$lib timeout 150 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$lib cfg5', d['ms_per_step'], 'attn', round(k['attention'],3), 'clk', d['clocks']['sm_mhz'])"
  ELIS_LIB=$lib timeout 100 python bench.py --workload cfg2 --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$lib cfg2', d['ms_per_step'], 'attn', round(k['attention'],3), 'clk', d['clocks']['sm_mhz'])"
done
done 2>&1 | tee gpurun_out/r02zk_ab_warp_issue.txt
ELIS_LIB=libelis.so timeout 200 python scripts/small_predict_latency.py --ns 4,64 --iters 100

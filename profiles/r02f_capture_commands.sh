# round-2 final (session 3): final-state capture -- GPU tests, smoke, bench lines (cfg5 default, reference arm, cfg2, cfg1,
# cfg3, one rank's cfg5 share), ncu launch list of the cfg5 step and --set full of its kernels
set -x
export PATH=/usr/local/cuda/bin:$PATH
for lib in libelis_wi0.so libelis.so; do
  ELIS_LIB=$lib timeout 90 python scripts/run_predict.py --n 256 --iters 1 --dump /tmp/cfg2_$lib.npz | tail -1
  ELIS_LIB=$lib timeout 90 python scripts/run_predict.py --workload cfg5 --iters 1 --dump /tmp/cfg5_$lib.npz | tail -1
done
python - <<'PY' 2>&1 | tee gpurun_out/r02f_warp_issue_bitwise.txt
import numpy as np
for w in ("cfg2", "cfg5"):
    a, b = np.load(f"/tmp/{w}_libelis_wi0.so.npz"), np.load(f"/tmp/{w}_libelis.so.npz")
    print(w, "attention thread-0 vs warp-elect MMA issue: pred bitwise equal:", np.array_equal(a["pred"].view(np.uint32), b["pred"].view(np.uint32)),
          "hidden bitwise equal:", np.array_equal(a["hidden"].view(np.uint32), b["hidden"].view(np.uint32)))
PY
timeout 200 python scripts/small_predict_latency.py --ns 1,4,16,64,256 --iters 100 > gpurun_out/r02f_small_predict.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02f_gpu_tests.log 2>&1; tail -2 gpurun_out/r02f_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; tail -1 gpurun_out/r02f_smoke.log
timeout 400 python bench.py > gpurun_out/r02f_bench_default.json 2> gpurun_out/r02f_bench.err
timeout 400 python bench.py --impl reference > gpurun_out/r02f_bench_ref.json 2>> gpurun_out/r02f_bench.err
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/r02f_bench_cfg2.json 2>> gpurun_out/r02f_bench.err
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline > gpurun_out/r02f_bench_cfg1.json 2>> gpurun_out/r02f_bench.err
timeout 600 python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_bench_cfg3.json 2>> gpurun_out/r02f_bench.err
timeout 300 python bench.py --requests 164 --no-cpu-baseline > gpurun_out/r02f_bench_cfg5_due164.json 2>> gpurun_out/r02f_bench.err
timeout 300 python bench.py --precision fp8 --no-cpu-baseline > gpurun_out/r02f_bench_cfg5_fp8.json 2>> gpurun_out/r02f_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches.csv \
  python scripts/run_predict.py --workload cfg5 --iters 2 > gpurun_out/r02f_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_attention_tc" -s 5 -c 5 \
  -o gpurun_out/r02f_full -f python scripts/run_predict.py --workload cfg5 --iters 1 > gpurun_out/r02f_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_embed_ln|k_pool|k_fc_tf32|k_head_out|k_make_keys|k_select_cluster|k_meta" -c 8 \
  -o gpurun_out/r02f_small -f python scripts/run_predict.py --workload cfg5 --iters 1 > gpurun_out/r02f_ncu_small.log 2>&1
ls -la gpurun_out/ | grep r02f

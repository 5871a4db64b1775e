# round-2b: cfg5 default bench (N=1), reference arm, cfg2, ncu launch list + --set full of window 0's layer-1 kernels
set -x
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02b_gpu_tests.log 2>&1; tail -3 gpurun_out/r02b_gpu_tests.log
timeout 300 python bench.py > gpurun_out/r02b_bench_default.json 2> gpurun_out/r02b_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r02b_bench_ref.json 2>> gpurun_out/r02b_bench.err
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/r02b_bench_cfg2.json 2>> gpurun_out/r02b_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches.csv \
  python scripts/run_predict.py --workload cfg5 --iters 2 > gpurun_out/r02b_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_attention_tc" -s 5 -c 5 \
  -o gpurun_out/r02b_full -f python scripts/run_predict.py --workload cfg5 --iters 1 > gpurun_out/r02b_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_embed_ln|k_pool|k_fc_f32|k_head_out|k_make_keys|k_select_topk" -c 6 \
  -o gpurun_out/r02b_small -f python scripts/run_predict.py --workload cfg5 --iters 1 > gpurun_out/r02b_ncu_small.log 2>&1
ls -la gpurun_out/

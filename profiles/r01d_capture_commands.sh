# round-1d profile capture (default path: fp16 operands + fp16 residual stream): launch list of the
# bench command, ncu --set full of one launch per GEMM / attention / head-FC kernel, bench lines
set -x
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01d_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r01d_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_attention_tc|k_fc_f32|k_pool|k_embed" -s 7 -c 9 \
  -o gpurun_out/r01d_full -f python scripts/run_predict.py --precision fp16 --residual16 --iters 1 > gpurun_out/r01d_ncu_full.log 2>&1
timeout 300 python bench.py > gpurun_out/r01d_bench_default.json 2> gpurun_out/r01d_bench.err
timeout 300 python bench.py --residual fp32 --no-cpu-baseline > gpurun_out/r01d_bench_fp16_res32.json 2>> gpurun_out/r01d_bench.err
timeout 300 python bench.py --precision bf16 --no-cpu-baseline > gpurun_out/r01d_bench_bf16.json 2>> gpurun_out/r01d_bench.err
timeout 300 python bench.py --precision fp8 --no-cpu-baseline > gpurun_out/r01d_bench_fp8.json 2>> gpurun_out/r01d_bench.err
timeout 300 python bench.py --pooling cls --cls-last-layer --no-cpu-baseline > gpurun_out/r01d_bench_cls_pruned.json 2>> gpurun_out/r01d_bench.err
timeout 300 python bench.py --config tiny --n 16 --lengths fixed:64 --no-cpu-baseline > gpurun_out/r01d_bench_tiny.json 2>> gpurun_out/r01d_bench.err
timeout 600 python bench.py --config large --n 4096 --lengths uniform --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01d_bench_large.json 2>> gpurun_out/r01d_bench.err
timeout 300 python bench.py --inflight 65536 --n 256 --no-cpu-baseline > gpurun_out/r01d_bench_inflight.json 2>> gpurun_out/r01d_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01d_bench_ref.json 2>> gpurun_out/r01d_bench.err
timeout 300 python scripts/select_latency.py > gpurun_out/r01d_select_latency.json 2>> gpurun_out/r01d_bench.err

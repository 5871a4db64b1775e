# round-1c profile capture (fp16 default path): launch list of the bench command, ncu --set full of
# layer-1 GEMM/attention launches, bench lines for the variants
set -x
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01c_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r01c_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_attention_tc" -s 5 -c 5 \
  -o gpurun_out/r01c_full -f python scripts/run_predict.py --precision fp16 --iters 1 > gpurun_out/r01c_ncu_full.log 2>&1
timeout 300 python bench.py > gpurun_out/r01c_bench_fp16.json 2> gpurun_out/r01c_bench.err
timeout 300 python bench.py --pooling cls --no-cpu-baseline > gpurun_out/r01c_bench_cls.json 2>> gpurun_out/r01c_bench.err
timeout 300 python bench.py --pooling cls --cls-last-layer --no-cpu-baseline > gpurun_out/r01c_bench_cls_pruned.json 2>> gpurun_out/r01c_bench.err
timeout 300 python bench.py --precision fp8 --no-cpu-baseline > gpurun_out/r01c_bench_fp8.json 2>> gpurun_out/r01c_bench.err
timeout 300 python bench.py --precision bf16 --no-cpu-baseline > gpurun_out/r01c_bench_bf16.json 2>> gpurun_out/r01c_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01c_bench_ref.json 2>> gpurun_out/r01c_bench.err

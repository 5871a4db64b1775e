# round-1f: after the st.async LN statistics exchange: launch list, ncu --set full of the layer-1 GEMM / attention launches, bench lines
set -x
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01f_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --graph off > gpurun_out/r01f_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_attention_tc" -s 6 -c 5 \
  -o gpurun_out/r01f_full -f python scripts/run_predict.py --precision fp16 --residual16 --iters 1 > gpurun_out/r01f_ncu_full.log 2>&1
timeout 300 python bench.py > gpurun_out/r01f_bench_default.json 2> gpurun_out/r01f_bench.err
timeout 300 python bench.py --graph off --no-cpu-baseline > gpurun_out/r01f_bench_eager.json 2>> gpurun_out/r01f_bench.err
timeout 300 python bench.py --residual fp32 --no-cpu-baseline > gpurun_out/r01f_bench_fp16_res32.json 2>> gpurun_out/r01f_bench.err
timeout 300 python bench.py --precision bf16 --no-cpu-baseline > gpurun_out/r01f_bench_bf16.json 2>> gpurun_out/r01f_bench.err
timeout 300 python bench.py --precision fp8 --no-cpu-baseline > gpurun_out/r01f_bench_fp8.json 2>> gpurun_out/r01f_bench.err
timeout 300 python bench.py --pooling cls --cls-last-layer --no-cpu-baseline > gpurun_out/r01f_bench_cls_pruned.json 2>> gpurun_out/r01f_bench.err
timeout 300 python bench.py --config tiny --requests 16 --lengths fixed:64 --no-cpu-baseline > gpurun_out/r01f_bench_tiny.json 2>> gpurun_out/r01f_bench.err
timeout 600 python bench.py --config large --requests 4096 --lengths uniform --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01f_bench_large.json 2>> gpurun_out/r01f_bench.err
timeout 300 python bench.py --inflight 65536 --requests 256 --no-cpu-baseline > gpurun_out/r01f_bench_inflight.json 2>> gpurun_out/r01f_bench.err
timeout 300 python bench.py --inflight 65536 --requests 164 --no-cpu-baseline > gpurun_out/r01f_bench_inflight_due164.json 2>> gpurun_out/r01f_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01f_bench_ref.json 2>> gpurun_out/r01f_bench.err

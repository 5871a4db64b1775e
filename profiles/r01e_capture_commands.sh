# round-1e: bench lines after CUDA-graph replay in bench.py (kernels as in r01d, whose ncu captures stand)
set -x
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01e_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --graph off > gpurun_out/r01e_ncu_bench.log 2>&1
timeout 300 python bench.py > gpurun_out/r01e_bench_default.json 2> gpurun_out/r01e_bench.err
timeout 300 python bench.py --graph off --no-cpu-baseline > gpurun_out/r01e_bench_eager.json 2>> gpurun_out/r01e_bench.err
timeout 300 python bench.py --residual fp32 --no-cpu-baseline > gpurun_out/r01e_bench_fp16_res32.json 2>> gpurun_out/r01e_bench.err
timeout 300 python bench.py --precision bf16 --no-cpu-baseline > gpurun_out/r01e_bench_bf16.json 2>> gpurun_out/r01e_bench.err
timeout 300 python bench.py --precision fp8 --no-cpu-baseline > gpurun_out/r01e_bench_fp8.json 2>> gpurun_out/r01e_bench.err
timeout 300 python bench.py --pooling cls --cls-last-layer --no-cpu-baseline > gpurun_out/r01e_bench_cls_pruned.json 2>> gpurun_out/r01e_bench.err
timeout 300 python bench.py --config tiny --requests 16 --lengths fixed:64 --no-cpu-baseline > gpurun_out/r01e_bench_tiny.json 2>> gpurun_out/r01e_bench.err
timeout 600 python bench.py --config large --requests 4096 --lengths uniform --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01e_bench_large.json 2>> gpurun_out/r01e_bench.err
timeout 300 python bench.py --inflight 65536 --requests 256 --no-cpu-baseline > gpurun_out/r01e_bench_inflight.json 2>> gpurun_out/r01e_bench.err
timeout 300 python bench.py --inflight 65536 --requests 164 --no-cpu-baseline > gpurun_out/r01e_bench_inflight_due164.json 2>> gpurun_out/r01e_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01e_bench_ref.json 2>> gpurun_out/r01e_bench.err

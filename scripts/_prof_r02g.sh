# round-2 final commit: GPU suite + smoke + bench lines (cfg5 default, reference arm, cfg1, cfg2, 164-due share)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02g_gpu_tests.log 2>&1; tail -2 gpurun_out/r02g_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; tail -1 gpurun_out/r02g_smoke.log
timeout 400 python bench.py > gpurun_out/r02g_bench_default.json 2> gpurun_out/r02g_bench.err
timeout 400 python bench.py --impl reference > gpurun_out/r02g_bench_ref.json 2>> gpurun_out/r02g_bench.err
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/r02g_bench_cfg2.json 2>> gpurun_out/r02g_bench.err
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline > gpurun_out/r02g_bench_cfg1.json 2>> gpurun_out/r02g_bench.err
timeout 300 python bench.py --requests 164 --no-cpu-baseline > gpurun_out/r02g_bench_cfg5_due164.json 2>> gpurun_out/r02g_bench.err
timeout 200 python scripts/small_predict_latency.py --ns 1,4,16,64,256 --iters 100 > gpurun_out/r02g_small_predict.jsonl 2>&1
ls gpurun_out | grep r02g

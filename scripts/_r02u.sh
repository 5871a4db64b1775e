# round-2 re-entry check: full GPU suite + smoke + default bench on the committed state
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02u_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02u_smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/r02u_bench_default.json 2> gpurun_out/r02u_bench_default.err
tail -3 gpurun_out/r02u_gpu_tests.txt; tail -1 gpurun_out/r02u_smoke.log; tail -c 600 gpurun_out/r02u_bench_default.json

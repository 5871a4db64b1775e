for sm in 0 1; do ELIS_GEMM_SMALLM=$sm timeout 200 python scripts/small_predict_latency.py --ns 1,4,16,64 --iters 100 | sed "s/^/smallm=$sm /"; done 2>&1 | tee gpurun_out/r02zt_small_predict.txt
timeout 900 python -m pytest tests/test_gpu_predict.py tests/test_gpu_residual16.py tests/test_gpu_graph.py -q -x 2>&1 | tail -2

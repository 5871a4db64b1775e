set -x
timeout 600 python -m pytest tests/test_gpu_graph.py -q -x > gpurun_out/r02p_graph.log 2>&1; tail -3 gpurun_out/r02p_graph.log; grep -E "Error|assert" gpurun_out/r02p_graph.log | head -10
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02p_gpu_tests.log 2>&1; tail -3 gpurun_out/r02p_gpu_tests.log; grep -E "^FAILED|Error" gpurun_out/r02p_gpu_tests.log | head

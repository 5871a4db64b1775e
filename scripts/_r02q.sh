set -x
timeout 900 python -m pytest tests/test_gpu_streamsim.py tests/test_gpu_arena.py -q -x > gpurun_out/r02q_tests.log 2>&1; tail -3 gpurun_out/r02q_tests.log; grep -E "Error|assert" gpurun_out/r02q_tests.log | head
timeout 2400 python scripts/run_streamsim.py --n 2000 --mults 0.7,0.9,3 --workers 1,8 > gpurun_out/r02q_streamsim.jsonl 2> gpurun_out/r02q_streamsim.err
tail -2 gpurun_out/r02q_streamsim.err
python - <<'PY'
import json
for l in open("gpurun_out/r02q_streamsim.jsonl"):
    d = json.loads(l)
    r = d["results"]
    print(d["workers"], d["rate_multiple"], {k: round(v["mean_jct_ms"]) for k, v in r.items()},
          "gpu ms/iter", round(r["isrtf_gpu"]["gpu_ms_per_iter"], 3), "host", round(r["isrtf_gpu"]["host_ms_per_iter"], 3), "due", round(r["isrtf_gpu"]["due_per_iter"],2))
PY

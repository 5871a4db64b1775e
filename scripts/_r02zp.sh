# cfg4 stream simulator on the final build: per-iteration GPU time with PDL + graph
timeout 1500 python scripts/run_streamsim.py --n 2000 --mults 0.7,0.9 --workers 1,8 --sources fcfs,isrtf_gpu,isrtf_oracle > gpurun_out/r02zp_streamsim.jsonl 2> gpurun_out/r02zp_streamsim.err
tail -2 gpurun_out/r02zp_streamsim.err
python - <<'PY'
import json
for l in open("gpurun_out/r02zp_streamsim.jsonl"):
    d = json.loads(l)
    r = d["results"]
    print(d["workers"], d["rate_multiple"], {k: round(v["mean_jct_ms"]) for k, v in r.items()},
          "gpu ms/iter", round(r["isrtf_gpu"]["gpu_ms_per_iter"], 3), "host", round(r["isrtf_gpu"]["host_ms_per_iter"], 3), "due", round(r["isrtf_gpu"]["due_per_iter"], 2))
PY

# small due sets (cfg4 regime): predict latency eager / graph, PDL on vs off
for p in 1 0 1 0; do ELIS_PDL=$p timeout 300 python scripts/small_predict_latency.py --ns 1,4,16,64,256; done 2>&1 | grep "^{" | tee gpurun_out/r02zf_small_predict.jsonl
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02zf_launches_n4.csv python scripts/small_predict_latency.py --ns 4 --iters 1 > /dev/null 2>&1; echo ncu rc=$?

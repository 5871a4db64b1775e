# round-2i: ncu of the 3xTF32 head layer at n = 1311 (cfg5 window) and n = 164 (one rank's share)
set -x
export PATH=/usr/local/cuda/bin:$PATH
timeout 300 ncu --set full --clock-control none -k regex:"k_fc_tf32" -s 1 -c 1 -o gpurun_out/r02i_fc1311 -f python scripts/run_predict.py --workload cfg5 --iters 1 > gpurun_out/r02i_ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"k_fc_tf32" -s 1 -c 1 -o gpurun_out/r02i_fc164 -f python scripts/run_predict.py --config base --n 164 --iters 1 > gpurun_out/r02i_ncu2.log 2>&1
ls gpurun_out/r02i*

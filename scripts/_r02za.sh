export ELIS_ATTN_ENGINE=66
ELIS_LIB=libelis_adbg.so timeout 120 python scripts/attn_repro.py trace:256 > gpurun_out/r02za_dbg.txt 2>&1
grep stuck gpurun_out/r02za_dbg.txt | wc -l
grep stuck gpurun_out/r02za_dbg.txt | awk '{print $7, $9, $11}' | sort | uniq -c | sort -rn | head -20
grep stuck gpurun_out/r02za_dbg.txt | head -20
tail -2 gpurun_out/r02za_dbg.txt

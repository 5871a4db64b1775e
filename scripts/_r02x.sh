for L in 64 1 65 "1,2" "1,2,63,64,65,130,7,512,200,33"; do
  ELIS_LIB=libelis_adbg.so timeout 60 python scripts/attn_repro.py $L 2>&1 | grep -v Warn | tail -4
  ELIS_PDL=0 ELIS_LIB=libelis_adbg.so timeout 60 python scripts/attn_repro.py $L 2>&1 | grep -v Warn | tail -2
done

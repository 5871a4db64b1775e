export ELIS_ATTN_ENGINE=66
run() { timeout 20 python scripts/attn_repro.py "$@" 2>&1 | grep -E "^ok|Error" | tail -1 | cut -c1-60 || true; }
L200=$(python -c "print(','.join(['200']*40))")
for i in 1 2 3; do echo "40x200 #$i: $(run $L200)"; done
for i in 1 2; do echo "trace:64 #$i: $(run trace:64)"; echo "trace:256 #$i: $(run trace:256)"; echo "trace:1311 #$i: $(run trace:1311)"; done
